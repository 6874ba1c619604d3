"""Multi-process (world_size 2, gloo, CPU) check of the data-parallel update
semantics the B200 path implements with NCCL: rank r runs worker r's batch
(train.cpp:232), scales its gradient by tokens_r/total before the sum
(train.cpp:254-269) and every rank applies the same Adam step.  Gradients come
from the unmodified reference (oracle/_ref); the result must equal the
reference's own threaded 2-worker trainSync update."""
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

    from paper_1804_00344_b200 import synth
    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank,
                            world_size=world)
    src, tgt = synth.corpus(12, 40)
    ex = R.Examples(src, tgt)
    bs = R.BatchSet(ex, BUDGET, 1)
    batches = R.make_batches(ex, BUDGET, 1)
    tokens = [float(b["tgt_mask"].sum()) for b in batches[:world]]
    total = np.float32(sum(np.float32(t) for t in tokens))
    model = R.RefModel(CFG, 1)
    mine = S.shard(take=world, world=world, local_workers=1, rank=rank)
    assert mine == [rank]
    _, tok = model.loss_grads(bs, rank, S.mix_seed(1, 0, rank))
    assert tok == tokens[rank]
    w = np.float32(np.float32(tok) / total)
    for n in model.param_names():
        g = torch.from_numpy(model.grad(n) * w)
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
