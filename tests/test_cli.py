"""`mtk-b200` command line: the reference's `mtk vocab|train` (tools/mtk.cpp)
on the B200 backend -- option names, config files, exit codes (0 ok,
1 usage, 2 data/io, 3 numeric), vocabulary order, and a training run whose
saved model matches the reference's trainSync on the same text corpus."""
import os
import subprocess
from collections import Counter

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_1804_00344_b200", "mtk-b200")


def run(*args, env=None):
    return subprocess.run([EXE, *args], capture_output=True, text=True, env=env)


def write(path, lines):
    path.write_text("".join(line + "\n" for line in lines))
    return str(path)


def test_cli_usage_and_data_errors(tmp_path):
    assert run().returncode == 1
    assert run("translate").returncode == 1            # missing required options
    assert run("train", "--model", "m").returncode == 1  # missing required options
    assert run("train", "--bogus", "1").returncode == 1
    r = run("vocab", "--corpus", str(tmp_path / "missing.txt"), "--output", str(tmp_path / "v"))
    assert r.returncode == 2 and "io error" in r.stderr
    empty = write(tmp_path / "empty.txt", [""])
    r = run("vocab", "--corpus", empty, "--output", str(tmp_path / "v"))
    assert r.returncode == 2 and "empty corpus" in r.stderr
    cfg = write(tmp_path / "bad.cfg", ["no-such-option: 3"])
    r = run("vocab", "--corpus", empty, "--output", str(tmp_path / "v"), "--config", cfg)
    assert r.returncode == 2


def test_cli_vocab_matches_reference_order(tmp_path):
    """data.cpp:34-61: </s>, <unk>, then descending frequency, ties
    lexicographic, truncated at --max-size (from a config file)."""
    lines = ["b a c a", "c c d e", "a e f"]
    corpus = write(tmp_path / "c.txt", lines)
    cfg = write(tmp_path / "v.cfg", ["# options", "max-size: 6"])
    out = tmp_path / "v.txt"
    r = run("vocab", "--corpus", corpus, "--output", str(out), "--config", cfg)
    assert r.returncode == 0, r.stderr
    freq = Counter(t for line in lines for t in line.split())
    order = sorted(freq, key=lambda t: (-freq[t], t))
    assert out.read_text().split("\n")[:-1] == ["</s>", "<unk>"] + order[:4]


@pytest.mark.gpu
def test_cli_train_matches_reference(cuda, tmp_path):
    """A short Transformer training run from text files: the saved model
    equals the reference trainSync on the same corpus within the DP
    tolerance (test_train.cpp:237-242), and a checkpoint is written."""
    from oracle import refbind as R
    from paper_1804_00344_b200 import config_text, mtk as M, synth
    V = 60
    src, tgt = synth.corpus(40, V)
    tok = lambda ids: " ".join(f"w{int(i)}" for i in ids)
    s_path = write(tmp_path / "s.txt", [tok(s) for s in src])
    t_path = write(tmp_path / "t.txt", [tok(t) for t in tgt])
    vocab = write(tmp_path / "vocab.txt", ["</s>", "<unk>"] + [f"w{i}" for i in range(2, V)])
    cfg = write(tmp_path / "train.cfg", ["arch: transformer", "emb-dim: 32", "heads: 2",
                                        "layers: 1", "dropout: 0", "tying: all",
                                        "mini-batch-tokens: 330", "max-updates: 2",
                                        "workers: 2", "save-every: 1", "seed: 9"])
    model = str(tmp_path / "model.mtk")
    env = dict(os.environ, MTK_PRECISION="fp32")
    r = run("train", "--model", model, "--train-sets", s_path, t_path, "--vocabs", vocab, vocab,
            "--config", cfg, env=env)
    assert r.returncode == 0, r.stderr
    assert "finished: updates=2" in r.stderr
    assert os.path.exists(model + ".ckpt") and os.path.exists(model + ".avg")
    ref_cfg = config_text(arch="transformer", vocab=V, emb=32, heads=2, layers=1, dropout=0.0,
                          tying="all")
    ref = R.RefModel(ref_cfg, 9)
    ref.train(R.Examples(src, tgt), workers=2, budget=330, seed=9, epochs=1, max_updates=2)
    g = M.ExpressionGraph(1)
    M.Model(M.read_model_config(model)).register_params(g)
    M.load_params(model, g)
    for n in ref.param_names():
        a, b = g.param_value(n), ref.param(n)
        assert np.allclose(a, b, rtol=1e-6, atol=1e-6 * max(1.0, np.abs(b).max())), n


@pytest.mark.gpu
def test_cli_train_async_matches_reference(cuda, tmp_path):
    """`train --async` with one worker (trainAsync, train.cpp:302-404) saves
    the same model as the reference's asynchronous run."""
    from oracle import refbind as R
    from paper_1804_00344_b200 import config_text, mtk as M, synth
    V = 60
    src, tgt = synth.corpus(40, V)
    tok = lambda ids: " ".join(f"w{int(i)}" for i in ids)
    s_path = write(tmp_path / "s.txt", [tok(s) for s in src])
    t_path = write(tmp_path / "t.txt", [tok(t) for t in tgt])
    vocab = write(tmp_path / "vocab.txt", ["</s>", "<unk>"] + [f"w{i}" for i in range(2, V)])
    cfg = write(tmp_path / "train.cfg", ["arch: transformer", "emb-dim: 32", "heads: 2",
                                        "layers: 1", "dropout: 0", "tying: all",
                                        "mini-batch-tokens: 330", "max-updates: 3",
                                        "workers: 1", "seed: 9"])
    model = str(tmp_path / "model.mtk")
    env = dict(os.environ, MTK_PRECISION="fp32")
    r = run("train", "--model", model, "--train-sets", s_path, t_path, "--vocabs", vocab, vocab,
            "--config", cfg, "--async", env=env)
    assert r.returncode == 0, r.stderr
    ref_cfg = config_text(arch="transformer", vocab=V, emb=32, heads=2, layers=1, dropout=0.0,
                          tying="all")
    ref = R.RefModel(ref_cfg, 9)
    ref.train(R.Examples(src, tgt), workers=1, budget=330, seed=9, epochs=1, max_updates=3,
              async_=True)
    g = M.ExpressionGraph(1)
    M.Model(M.read_model_config(model)).register_params(g)
    M.load_params(model, g)
    for n in ref.param_names():
        a, b = g.param_value(n), ref.param(n)
        assert np.allclose(a, b, rtol=1e-6, atol=1e-6 * max(1.0, np.abs(b).max())), n


@pytest.mark.gpu
def test_cli_translate_and_score(cuda, tmp_path):
    """`translate` (beam search, n-best file in the reference's
    "id ||| text ||| F0=... ||| score" format) and `score` (forced decoding)
    on a model trained by `train`; outputs agree with the Python API
    (beam_search / score_batch, themselves pinned to the reference in
    tests/test_search_gpu.py)."""
    from paper_1804_00344_b200 import mtk as M, synth
    V = 40
    src, tgt = synth.corpus(24, V)
    tok = lambda ids: " ".join(f"w{int(i)}" for i in ids)
    s_path = write(tmp_path / "s.txt", [tok(s) for s in src])
    t_path = write(tmp_path / "t.txt", [tok(t) for t in tgt])
    vocab = write(tmp_path / "vocab.txt", ["</s>", "<unk>"] + [f"w{i}" for i in range(2, V)])
    model = str(tmp_path / "model.mtk")
    env = dict(os.environ, MTK_PRECISION="fp32")
    r = run("train", "--model", model, "--train-sets", s_path, t_path, "--vocabs", vocab, vocab,
            "--arch", "transformer", "--emb-dim", "32", "--heads", "2", "--layers", "1",
            "--dropout", "0", "--tying", "all", "--max-updates", "20", "--lr", "0.01",
            "--warmup", "1", "--mini-batch-tokens", "400", "--quiet", env=env)
    assert r.returncode == 0, r.stderr
    out, nb = tmp_path / "out.txt", tmp_path / "nbest.txt"
    r = run("translate", "--models", model, "--vocabs", vocab, vocab, "--input", s_path,
            "--output", str(out), "--n-best-file", str(nb), "--n-best", "2", "--beam-size", "3",
            "--mini-batch-tokens", "4096", env=env)
    assert r.returncode == 0, r.stderr
    best = out.read_text().split("\n")[:-1]
    assert len(best) == len(src)
    lines = nb.read_text().split("\n")[:-1]
    assert all(len(ln.split(" ||| ")) == 4 and " F0=" in ln for ln in lines)
    r = run("score", "--model", model, "--vocabs", vocab, vocab, "--input", s_path, t_path,
            "--output", str(tmp_path / "scores.txt"), env=env)
    assert r.returncode == 0, r.stderr
    scores = [float(ln.split()[1]) for ln in (tmp_path / "scores.txt").read_text().split("\n")[:-1]]
    assert len(scores) == len(src)

    M.set_precision("fp32")
    try:
        m = M.Model(M.read_model_config(model))
        g = M.ExpressionGraph(1)
        m.register_params(g)
        M.load_params(model, g)
        ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
        for b in M.make_batches(ex, 100000, 1, False):
            ids = b.sentence_ids()
            hyps = M.beam_search(m, g, b, beam=3, alpha=0.6, max_length_factor=3)
            sc = M.score_batch(m, g, b)
            for r_, sid in enumerate(ids):
                toks = [t for t in hyps[r_][0][0] if t != 0]
                assert best[sid] == tok(toks), sid
                assert abs(scores[sid] - sc[r_][1]) <= 1e-5 * max(1.0, abs(sc[r_][1])), sid
    finally:
        M.set_precision("tf32")
