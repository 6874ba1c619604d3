"""Drop-in proof: the reference's UNMODIFIED model code on this backend.

tests/dropin/_build/dropin_step links the reference's own src/models.cpp,
src/layers.cpp and src/encdec.cpp -- compiled from /root/reference against
this build's headers (csrc/host/mtk/*.h; tests/dropin/Makefile) -- with
libmtkhost.so / libmtkcuda.so, and runs buildModel -> registerParams ->
buildLoss -> forward -> backward (the reference's trainSync call sequence,
train.cpp:232-235).  Its loss and every parameter gradient must match the
reference oracle (oracle/_ref) at the FP32 step tolerances
(tests/parity_util.py): the ExpressionGraph surface (graph.h:60-127) and the
Encoder/Decoder interfaces are source- and behaviour-compatible.

The reference layers use the generic ops (dot, softmax, add, gruCell, ...),
not this build's fused nodes, so this also covers the unfused op paths at
model scale.
"""
import os
import struct
import subprocess

import numpy as np
import pytest

from oracle import refbind as R
from paper_1804_00344_b200 import config_text, synth
from parity_util import check_grads

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "dropin", "_build", "dropin_step")

CASES = {
    "transformer": dict(arch="transformer", vocab=600, emb=64, heads=4, layers=2),
    "s2s-shallow": dict(arch="s2s-shallow", vocab=300, emb=32, state=48),
    "s2s-deep-ln": dict(arch="s2s-deep", vocab=300, emb=32, state=48, layer_norm=True),
    # host dropout masks (the reference's draws; MTK_DROPOUT_RNG=host)
    "transformer-dropout": dict(arch="transformer", vocab=8000, emb=256, heads=4, layers=2,
                                dropout=0.1),
}


def read_out(path):
    with open(path, "rb") as f:
        loss, tok, n = struct.unpack("<dqq", f.read(24))
        grads = {}
        for _ in range(n):
            (ln,) = struct.unpack("<q", f.read(8))
            name = f.read(ln).decode()
            (cnt,) = struct.unpack("<q", f.read(8))
            grads[name] = np.frombuffer(f.read(4 * cnt), np.float32).copy()
    return loss, tok, grads


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
@pytest.mark.parametrize("name", list(CASES))
def test_reference_model_code_on_b200_backend(cuda, tmp_path, name, prec):
    if not os.path.exists(EXE):
        pytest.fail("tests/dropin/_build/dropin_step missing: run __graft_entry__.build() "
                    "where /root/reference exists")
    spec = CASES[name]
    cfg = config_text(**spec)
    n, seed = 12, 0x5EED
    cf = tmp_path / "model.cfg"
    cf.write_text(cfg)
    out = tmp_path / "grads.bin"
    env = dict(os.environ, MTK_PRECISION=prec, MTK_DROPOUT_RNG="host")
    r = subprocess.run([EXE, str(cf), str(n), str(n * 66), str(seed), str(out)], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr + r.stdout
    loss, tok, grads = read_out(out)

    src, tgt = synth.corpus(n, spec["vocab"])
    ref = R.RefModel(cfg, 1)
    bs = R.BatchSet(R.Examples(src, tgt), n * 66, 1)
    rloss, rtok = ref.loss_grads(bs, 0, seed)
    names = ref.param_names()
    assert list(grads) == names  # creation order and names
    assert tok == rtok
    tol = 1e-5 if prec == "fp32" else 2e-3
    assert abs(loss - rloss) <= tol * abs(rloss), (loss, rloss)
    ref_grads = {k: ref.grad(k) for k in names}
    mine = {k: grads[k].reshape(ref_grads[k].shape) for k in names}
    check_grads(names, mine, ref_grads, prec, f"dropin-{name}")
