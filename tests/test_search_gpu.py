"""Decoding on the device: beam search and forced-decoding
scores vs the reference's search.cpp on the same trained model file and the
same batch.  FP32 mode; n-best token sequences identical, scores within 1e-6
relative (the log-softmax and ranking run on the host in double precision,
like the reference)."""
import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import config_text, mtk as M, synth

pytestmark = pytest.mark.gpu

V = 40


@pytest.fixture(autouse=True)
def fp32_mode(cuda):
    M.set_precision("fp32")
    yield
    M.set_precision("tf32")


def _trained_pair(cfg, tmp_path):
    src, tgt = synth.corpus(48, V)
    ref = R.RefModel(cfg, 11)
    ref.train(R.Examples(src, tgt), workers=1, budget=8 * 66, seed=11, epochs=3, max_updates=24,
              lr_base=0.01, warmup=1)
    path = str(tmp_path / "m.mtk")
    ref.save_model(path)
    model = M.Model(cfg)
    g = M.ExpressionGraph(1)
    model.register_params(g)
    M.load_params(path, g)
    return src, tgt, ref, model, g


@pytest.mark.parametrize("arch,ln", [("transformer", False), ("s2s-shallow", False),
                                     ("s2s-deep", True)])
def test_beam_search_and_scores_match_reference(tmp_path, arch, ln):
    cfg = config_text(arch=arch, vocab=V, emb=32, state=48, heads=2, layers=1, dropout=0.0,
                      tying="all", layer_norm=ln)
    src, tgt, ref, model, g = _trained_pair(cfg, tmp_path)
    n = 6
    ref_bs = R.BatchSet(R.Examples(src[:n], tgt[:n]), n * 66, 1, False)
    ours_b = M.make_batches(M.Examples([list(map(int, s)) for s in src[:n]],
                                       [list(map(int, t)) for t in tgt[:n]]), n * 66, 1, False)
    assert ref_bs.count == 1 and len(ours_b) == 1
    rows = ours_b[0].rows()
    want = ref.beam_search(ref_bs, 0, rows, beam=3, alpha=0.6, len_factor=2)
    got = M.beam_search(model, g, ours_b[0], beam=3, alpha=0.6, max_length_factor=2)
    assert len(got) == len(want)
    for s in range(rows):
        assert [h[0] for h in got[s]] == [h[0] for h in want[s]], s
        for (gt, gs, _), (wt, ws) in zip(got[s], want[s]):
            assert abs(gs - ws) <= 1e-6 * max(1.0, abs(ws)), (s, gs, ws)
    want_sc = ref.score_batch(ref_bs, 0, rows)
    got_sc = np.array([h[1] for h in M.score_batch(model, g, ours_b[0])])
    np.testing.assert_allclose(got_sc, want_sc, rtol=1e-6, atol=1e-6)
