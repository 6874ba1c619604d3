"""MTK1 model files and checkpoint/resume (
reference: serialize.cpp:37-133, train.cpp:121-164, 284-287, 407-418).

* files are byte-identical to the reference's for the same parameters /
  optimizer state, and load in both directions bit-exactly;
* a checkpointed-and-resumed run equals the uninterrupted run bitwise
  (the reference's own acceptance test, test_train.cpp:245-289).
"""
import os

import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import config_text, mtk as M, synth

pytestmark = pytest.mark.gpu

CFG = config_text(arch="transformer", vocab=60, emb=32, heads=2, layers=1)


def _examples(n=40, seed_vocab=60):
    src, tgt = synth.corpus(n, seed_vocab)
    return src, tgt, M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])


def _opts(**kw):
    o = M.TrainOptions()
    o.workers = 1
    o.token_budget = 5 * 66
    o.seed = 3
    o.epochs = 100
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def test_model_file_roundtrip_with_reference(cuda, tmp_path):
    ref = R.RefModel(CFG, 5)
    ref_file = str(tmp_path / "ref.mtk")
    ref.save_model(ref_file)
    # ours loads the reference's file bit-exactly ...
    model = M.Model(CFG)
    g = M.ExpressionGraph(99)  # different init: the file must win
    model.register_params(g)
    M.load_params(ref_file, g)
    for n in ref.param_names():
        assert np.array_equal(g.param_value(n), ref.param(n)), n
    # ... and writes the same bytes back
    ours = str(tmp_path / "ours.mtk")
    M.save_model(ours, CFG, g)
    assert open(ours, "rb").read() == open(ref_file, "rb").read()
    assert M.read_model_config(ours) == M.read_model_config(ref_file)
    # the reference loads ours
    ref2 = R.RefModel(CFG, 77)
    ref2.load_params(ours)
    for n in ref.param_names():
        assert np.array_equal(ref2.param(n), ref.param(n)), n


def test_model_file_errors(cuda, tmp_path):
    bad = tmp_path / "bad.mtk"
    bad.write_bytes(b"XXXX")
    model = M.Model(CFG)
    g = M.ExpressionGraph(1)
    model.register_params(g)
    with pytest.raises(M.DataError):
        M.load_params(str(bad), g)
    good = str(tmp_path / "good.mtk")
    M.save_model(good, CFG, g)
    data = open(good, "rb").read()
    (tmp_path / "trunc.mtk").write_bytes(data[: len(data) // 2])
    with pytest.raises(M.IoError):
        M.load_params(str(tmp_path / "trunc.mtk"), g)
    other = M.Model(config_text(arch="transformer", vocab=60, emb=16, heads=2, layers=1))
    g2 = M.ExpressionGraph(1)
    other.register_params(g2)
    with pytest.raises(M.DataError):
        M.load_params(good, g2)


def test_checkpoint_state_matches_reference(cuda, tmp_path):
    """A checkpoint the reference writes after 3 updates loads here with
    every parameter, Adam moment, EMA value and counter bit-exact, and our
    re-save is byte-identical."""
    src, tgt, ex = _examples()
    ref = R.RefModel(CFG, 3)
    ck = str(tmp_path / "ref.ckpt")
    ref.train_ckpt(R.Examples(src, tgt), workers=1, budget=5 * 66, seed=3, epochs=100,
                   max_updates=3, checkpoint_path=ck, checkpoint_every=3)
    model = M.Model(CFG)
    g = M.ExpressionGraph(50)
    model.register_params(g)
    adam = M.Adam(M.adam_defaults_for(CFG))
    avg = M.AveragedParameters()
    counters = M.load_checkpoint(ck, g, adam, avg)
    assert counters == R.RefModel(CFG, 1).load_checkpoint(ck)
    assert adam.step() == ref.adam_step() == 3
    for n in ref.param_names():
        assert np.array_equal(g.param_value(n), ref.param(n)), n
        assert np.array_equal(adam.first_moment(g, n), ref.state("m", n)), n
        assert np.array_equal(adam.second_moment(g, n), ref.state("v", n)), n
        assert np.array_equal(avg.value(g, n), ref.state("avg", n)), n
    ours = str(tmp_path / "ours.ckpt")
    M.save_checkpoint(ours, CFG, g, adam, avg, *counters)
    assert open(ours, "rb").read() == open(ck, "rb").read()


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_resume_reproduces_uninterrupted_run_bitwise(cuda, tmp_path, prec):
    """test_train.cpp:245-289 on the B200 path: 20 updates straight vs 10,
    checkpoint, fresh objects with a different init seed, resume to 20."""
    M.set_precision(prec)
    try:
        _, _, ex = _examples()
        model = M.Model(CFG)
        gF, aF, vF = M.ExpressionGraph(3), M.Adam(), M.AveragedParameters()
        rF, _ = M.train(model, ex, gF, aF, vF, _opts(max_updates=20))
        ck = str(tmp_path / "half.ckpt")
        gH, aH, vH = M.ExpressionGraph(3), M.Adam(), M.AveragedParameters()
        M.train(model, ex, gH, aH, vH, _opts(max_updates=10, checkpoint_path=ck,
                                              checkpoint_every=10))
        assert os.path.exists(ck)
        gR, aR, vR = M.ExpressionGraph(3 + 77), M.Adam(), M.AveragedParameters()
        rR, _ = M.train(model, ex, gR, aR, vR, _opts(max_updates=20, resume_from=ck))
        assert rR.updates == rF.updates == 20
        assert aR.step() == aF.step() == 20
        for n in gF.param_names():
            assert np.array_equal(gF.param_value(n), gR.param_value(n)), n
            assert np.array_equal(vF.value(gF, n), vR.value(gR, n)), n
    finally:
        M.set_precision("tf32")
