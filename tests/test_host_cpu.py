"""CPU-side checks of the product: the C-ABI library loads and exports every
symbol its header declares, host-side batching is bit-exact with the
reference, and the host restatements (seeds, schedule, config text) agree
with the oracle.  No kernel is launched here (there is no GPU)."""
import ctypes
import subprocess

import numpy as np
import pytest

from oracle import refbind as R
from oracle import restate as S
from paper_1804_00344_b200 import cabi, mtk as M, synth


def test_cabi_exports_every_declared_symbol():
    lib = cabi.lib()
    names = cabi.declared_symbols()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_cabi_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", cabi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_tcgen05_in_sass():
    out = subprocess.run(["cuobjdump", "-sass", cabi.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in out.stdout and "UTMALDG" in out.stdout and "LDTM" in out.stdout


def test_synth_python_matches_cpp():
    src, tgt = synth.corpus(50, 32000, start=7)
    ex = M.synth_examples(50, 32000, 7)
    py = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
    a = M.make_batches(ex, 5000, 3, True)
    b = M.make_batches(py, 5000, 3, True)
    for x, y in zip(a, b):
        assert np.array_equal(x.src_ids(), y.src_ids()) and np.array_equal(x.tgt_ids(), y.tgt_ids())


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("budget,seed,n", [(64 * 66, 1, 64), (4224, 9, 500), (16384, 1, 2000),
                                           (300, 2, 200), (70, 5, 40)])
def test_batching_bitexact_vs_reference(budget, seed, n):
    """makeBatches (data.cpp:226-282): ids, masks, sentence order identical."""
    src, tgt = synth.corpus(n, 8000)
    mine = M.make_batches(M.Examples([list(map(int, s)) for s in src],
                                     [list(map(int, t)) for t in tgt]), budget, seed, True)
    ref = R.make_batches(R.Examples(src, tgt), budget, seed)
    assert len(mine) == len(ref)
    for a, b in zip(mine, ref):
        assert np.array_equal(a.src_ids(), b["src_ids"])
        assert np.array_equal(a.tgt_ids(), b["tgt_ids"])
        assert np.array_equal(a.src_mask(), b["src_mask"])
        assert np.array_equal(a.tgt_mask(), b["tgt_mask"])
        assert list(a.sentence_ids()) == list(b["sent_ids"])


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
def test_batching_edge_cases_vs_reference():
    """Empty sentences, over-budget sentences (skipped), no shuffle."""
    src = [[], [5, 6, 7], [3] * 40, [9], [4, 4]]
    tgt = [[2], [], [3] * 40, [8, 8, 8], []]
    for budget, shuffle in [(20, True), (20, False), (200, True)]:
        mine = M.make_batches(M.Examples(src, tgt), budget, 4, shuffle)
        ref = R.make_batches(R.Examples(src, tgt), budget, 4, shuffle)
        assert len(mine) == len(ref)
        for a, b in zip(mine, ref):
            assert np.array_equal(a.src_ids(), b["src_ids"])
            assert np.array_equal(a.tgt_mask(), b["tgt_mask"])


def test_batch_config1_shape():
    """Config 1: exactly one batch, B=64, S=T=33, 1619 tokens."""
    bs = M.make_batches(M.synth_examples(64, 8000), 64 * 66, 1, True)
    assert len(bs) == 1
    assert bs[0].src_ids().shape == (64, 33) and bs[0].tgt_ids().shape == (64, 33)
    assert bs[0].target_tokens() == 1619


def test_lr_schedule_matches_restatement():
    s = M.LrSchedule()
    for step in [0, 1, 17, 8000, 16000, 16001, 64000, 10 ** 6]:
        assert s(step) == S.lr_schedule(step), step


def test_mix_seed_matches_restatement():
    for seed, u, w in [(1, 0, 0), (5, 3, 2), (2 ** 40, 10 ** 6, 7)]:
        assert M.mix_seed(seed, u, w) == S.mix_seed(seed, u, w)


def test_model_config_round_trip_and_errors():
    text = ("architecture: s2s-deep\nsource-vocab: 50000\ntarget-vocab: 50000\nemb-dim: 512\n"
            "state-dim: 1024\nlayer-norm: 1\ntying: all\n")
    c = M.ModelConfig.parse(text)
    assert c.architecture == "s2s-deep" and c.layer_norm and c.state_dim == 1024
    assert M.ModelConfig.parse(c.serialize()).serialize() == c.serialize()
    with pytest.raises(M.DataError):
        M.ModelConfig.parse("bogus-key: 1\n")


def test_error_taxonomy():
    for e in (M.DimensionError, M.NumericError, M.ContractError, M.DataError, M.IoError):
        assert issubclass(e, M.Error)


def test_dp_sharding_restatement():
    # worker i = rank*L + j handles batch idx+i (train.cpp:232); idle ranks at the tail
    assert S.shard(take=8, world=4, local_workers=2, rank=3) == [6, 7]
    assert S.shard(take=5, world=4, local_workers=2, rank=3) == []
    assert S.shard(take=5, world=4, local_workers=2, rank=2) == [4]


def test_arena_enforces_capacity():
    """Arena capacity check (tensor.cpp:42-44; test_tensor.cpp:209-212): the
    request is refused with NumericError before any device memory is taken."""
    from paper_1804_00344_b200 import mtk as M
    a = M.Arena(64)
    with pytest.raises(M.NumericError):
        a.alloc(1000)
    assert a.outstanding_bytes() == 0
