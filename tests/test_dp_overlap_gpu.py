"""Bucketed gradient all-reduce overlapped with the backward sweep
(SyncStepper, TrainOptions.overlap_allreduce).

On one GPU a one-rank NCCL communicator (force_comm) runs the real exchange
path: bucket schedule from the graph's lowest-consumer indices, events from
the compute stream, all-reduces on the communication stream, compute waits
before Adam.  A one-rank all-reduce is the identity, so parameters after
several updates must equal the run without any exchange bitwise, for both
the overlapped (many buckets) and the single post-backward all-reduce.
"""
import numpy as np
import pytest

from paper_1804_00344_b200 import config_text, mtk as M, synth

pytestmark = pytest.mark.gpu

CFG = config_text(arch="transformer", vocab=300, emb=64, heads=4, layers=2)


def _run(mode):
    """mode: None (no communicator), 'overlap', 'single'."""
    if mode is None:
        M.set_distributed(0, 1, bytes(128), False)
    else:
        M.set_distributed(0, 1, bytes(M.nccl_unique_id()), True)
    model = M.Model(CFG)
    g = M.ExpressionGraph(4)
    model.register_params(g)
    g.clear()
    adam = M.Adam(M.adam_defaults_for(CFG))
    avg = M.AveragedParameters()
    opts = M.TrainOptions()
    opts.workers = 2  # two local workers: only the last one's backward exchanges
    opts.token_budget = 8 * 66
    opts.seed = 4
    opts.overlap_allreduce = mode == "overlap"
    opts.bucket_elems = 20000  # many buckets for a small model
    st = M.SyncStepper(model, g, adam, avg, opts)
    src, tgt = synth.corpus(64, 300)
    ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
    batches = M.make_batches(ex, 8 * 66, 1, True)
    losses = []
    for u in range(3):
        r = st.update(batches[2 * u:2 * u + 2], u, True)
        losses.append(r.loss)
    params = {n: g.param_value(n).copy() for n in g.param_names()}
    return losses, params, st.buckets_issued()


def test_overlapped_bucket_allreduce_is_exact(cuda):
    try:
        base_l, base_p, nb0 = _run(None)
        ov_l, ov_p, nb = _run("overlap")
        one_l, one_p, nb1 = _run("single")
    finally:
        M.set_distributed(0, 1, bytes(128), False)
    assert nb0 == 0 and nb1 == 0
    assert nb >= 3 * 4, "expected several buckets per update"
    assert base_l == ov_l == one_l
    for n in base_p:
        assert np.array_equal(base_p[n], ov_p[n]), n
        assert np.array_equal(base_p[n], one_p[n]), n
