"""Two ranks, one GPU each, through the product's SyncStepper and a real
two-rank NCCL communicator (skipped on boxes with fewer than 2 GPUs).

* world = 2 (rank r runs worker r, gradients pre-scaled by tokens_r/total and
  summed by the bucketed NCCL all-reduce overlapped with the backward) must
  equal the one-process two-worker update (train.cpp:221-272) within the
  reference's own DP tolerance (1e-6 relative, test_train.cpp:237-242);
* the epoch-tail update with one batch (rank 1 idle, contributing zero with
  the same bucket sequence) must equal the one-worker update;
* both replicas stay bitwise identical;
* bench.py --gpus 2 launches two ranks and reports n_gpus = nccl_ranks = 2.
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


need2 = pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs")

CFG = dict(arch="transformer", vocab=300, emb=64, heads=4, layers=2)


def _batches(M):
    from paper_1804_00344_b200 import synth
    src, tgt = synth.corpus(60, CFG["vocab"])
    ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
    return M.make_batches(ex, 8 * 66, 1, True)


def _run(rank, world, uid, out, overlap):
    sys.path.insert(0, ROOT)
    from paper_1804_00344_b200 import config_text, mtk as M
    M.select_device(rank)
    M.set_precision("fp32")
    if world > 1:
        M.set_distributed(rank, world, uid)
    cfg = config_text(**CFG)
    model = M.Model(cfg)
    g = M.ExpressionGraph(1)
    model.register_params(g)
    g.clear()
    adam = M.Adam(M.adam_defaults_for(cfg))
    avg = M.AveragedParameters()
    opts = M.TrainOptions()
    opts.workers = 2
    opts.overlap_allreduce = overlap
    opts.bucket_elems = 20000  # several buckets even for this small model
    st = M.SyncStepper(model, g, adam, avg, opts)
    b = _batches(M)
    losses = [st.update([b[0], b[1]], 0, True).loss,   # both workers
              st.update([b[2]], 1, True).loss]         # epoch tail: one batch
    np.savez(out, losses=np.array(losses), **{n: g.param_value(n) for n in g.param_names()})


def _rank_main(rank, world, uid, d, overlap):
    _run(rank, world, uid, os.path.join(d, f"r{rank}.npz"), overlap)


@need2
@pytest.mark.parametrize("overlap", [True, False])
def test_two_ranks_equal_one_process_two_workers(overlap):
    import torch.multiprocessing as mp
    from paper_1804_00344_b200 import mtk as M
    uid = bytes(M.nccl_unique_id())
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.get_context("spawn")
        ps = [ctx.Process(target=_rank_main, args=(r, 2, uid, d, overlap)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(600)
            assert p.exitcode == 0
        single = os.path.join(d, "single.npz")
        p = ctx.Process(target=_run, args=(0, 1, b"", single, overlap))
        p.start()
        p.join(600)
        assert p.exitcode == 0
        r0, r1, s1 = (np.load(os.path.join(d, f)) for f in ("r0.npz", "r1.npz", "single.npz"))
        assert np.allclose(r0["losses"], s1["losses"], rtol=1e-6)
        for n in s1.files:
            if n == "losses":
                continue
            assert np.array_equal(r0[n], r1[n]), n  # identical replicas
            assert np.allclose(r0[n], s1[n], rtol=1e-6, atol=1e-6 * max(1.0, np.abs(s1[n]).max())), n


@need2
def test_bench_two_gpus_reports_two_ranks():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config",
                        "tiny", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], cwd=ROOT,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 2 and d["nccl_ranks"] == 2 and d["value"] > 0
