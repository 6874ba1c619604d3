"""Multi-process (world_size 2, gloo, CPU) check of the data-parallel update
the B200 path runs with NCCL: every rank asks the PRODUCT's host planner
(`rankShare`, csrc/host/train.cpp, the function SyncStepper::update uses) which
workers it runs and with which weight (train.cpp:221-269), computes those
workers' gradients (the unmodified reference, oracle/_ref, stands in for the
device step on a CPU-only box), pre-scales them, sums them over ranks (gloo
all_reduce standing in for the NCCL bucket all-reduce) and applies the same
Adam step.  The result must equal the reference's own threaded 2-worker
trainSync update bitwise, and both replicas must stay identical."""
import os
import tempfile

import numpy as np
import pytest

from oracle import refbind as R
from oracle import restate as S

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")

CFG = ("architecture: transformer\nsource-vocab: 40\ntarget-vocab: 40\nemb-dim: 16\n"
       "heads: 2\nlayers: 1\ndropout: 0\ntying: all\n")
BUDGET = 3 * 66


def _worker(rank, world, init_file, out_dir):
    import torch
    import torch.distributed as dist

    from paper_1804_00344_b200 import mtk as M, synth
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    src, tgt = synth.corpus(12, 40)
    ex = R.Examples(src, tgt)
    bs = R.BatchSet(ex, BUDGET, 1)
    batches = R.make_batches(ex, BUDGET, 1)
    tokens = [float(b["tgt_mask"].sum()) for b in batches[:world]]
    total = np.float32(sum(np.float32(t) for t in tokens))
    model = R.RefModel(CFG, 1)
    share = M.rank_share(tokens, world, world, rank)  # the product's planner
    assert [i for i, _ in share] == [rank]
    acc = {n: np.zeros(model.shape(n), np.float32) for n in model.param_names()}
    for i, w in share:
        _, tok = model.loss_grads(bs, i, M.mix_seed(1, 0, i))
        assert tok == tokens[i]
        assert np.float32(w) == np.float32(np.float32(tok) / total)
        for n in acc:
            acc[n] = acc[n] + model.grad(n) * np.float32(w)
    for n in model.param_names():
        g = torch.from_numpy(acc[n])
        dist.all_reduce(g)  # sum over ranks (NCCL on the GPU path)
        model.set_grad(n, g.numpy())
    model.adam_update(float(S.lr_schedule(1)))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
             **{n: model.param(n) for n in model.param_names()})
    dist.destroy_process_group()


def test_two_rank_update_equals_reference_two_worker_train():
    import torch.multiprocessing as mp

    from paper_1804_00344_b200 import synth
    with tempfile.TemporaryDirectory() as d:
        init_file = os.path.join(d, "init")
        mp.spawn(_worker, args=(2, init_file, d), nprocs=2, join=True)
        r0 = np.load(os.path.join(d, "rank0.npz"))
        r1 = np.load(os.path.join(d, "rank1.npz"))
        src, tgt = synth.corpus(12, 40)
        ref = R.RefModel(CFG, 1)
        ref.train(R.Examples(src, tgt), workers=2, budget=BUDGET, seed=1, epochs=1,
                  max_updates=1)
        for n in ref.param_names():
            assert np.array_equal(r0[n], r1[n]), n  # replicas stay identical
            assert np.array_equal(r0[n], ref.param(n)), n


@pytest.mark.parametrize("take,workers,world", [(8, 8, 8), (5, 8, 8), (8, 8, 2), (3, 8, 2),
                                                (1, 2, 2), (4, 4, 1), (7, 16, 4)])
def test_rank_share_partitions_workers(take, workers, world):
    """rankShare: the ranks' worker sets partition 0..take-1 (worker i = rank*L + j,
    train.cpp:232), idle ranks at the epoch tail run none, and the weights are
    (Real)tokens_i / (Real)total (train.cpp:262-266)."""
    from paper_1804_00344_b200 import mtk as M
    tokens = [float(100 + 13 * i) for i in range(take)]
    total = sum(tokens)
    seen = []
    for r in range(world):
        share = M.rank_share(tokens, workers, world, r)
        assert [i for i, _ in share] == S.shard(take, world, workers // world, r)
        for i, w in share:
            assert np.float32(w) == np.float32(np.float32(tokens[i]) / np.float32(total))
        seen += [i for i, _ in share]
    assert sorted(seen) == list(range(take))


def test_rank_share_rejects_bad_layouts():
    from paper_1804_00344_b200 import mtk as M
    with pytest.raises(M.ContractError):
        M.rank_share([1.0, 2.0, 3.0], 3, 2, 0)  # workers not a multiple of the ranks
    with pytest.raises(M.ContractError):
        M.rank_share([1.0] * 5, 4, 2, 0)  # more batches than workers
    with pytest.raises(M.ContractError):
        M.rank_share([1.0], 2, 2, 2)  # rank outside the communicator
