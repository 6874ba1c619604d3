"""Loss of the RNN models vs the reference at several dimensions (FP32 and
TF32 GEMMs), to locate where the shallow model's loss deviates."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import refbind as R
from paper_1804_00344_b200 import config_text, mtk as M, synth

def mine(cfg, src, tgt, n, prec):
    M.set_precision(prec)
    ex = M.Examples([list(map(int, s)) for s in src], [list(map(int, t)) for t in tgt])
    b = M.make_batches(ex, n * 66, 1, True)[0]
    model = M.Model(cfg); g = M.ExpressionGraph(1); model.register_params(g); g.clear(); g.set_seed(1)
    loss = model.build_loss(g, b); g.forward()
    return float(loss.val()[0])

for arch, ln in [("s2s-shallow", False), ("s2s-deep", False), ("s2s-deep", True)]:
    for V, e, d, n in [(60, 16, 24, 2), (50000, 16, 24, 2), (60, 512, 1024, 2), (60, 512, 1024, 16)]:
        cfg = config_text(arch=arch, vocab=V, emb=e, state=d, layer_norm=ln)
        src, tgt = synth.corpus(n, V)
        t0 = time.time()
        ref = R.RefModel(cfg, 1)
        rl = ref.forward_loss(R.BatchSet(R.Examples(src, tgt), n * 66, 1), 0, 1)
        l32 = mine(cfg, src, tgt, n, "fp32"); ltf = mine(cfg, src, tgt, n, "tf32")
        print(f"{arch:12s} ln={int(ln)} V={V:5d} e={e:4d} d={d:5d} n={n:2d}: ref {rl:.7f} "
              f"fp32 rel {abs(l32-rl)/rl:.2e}  tf32 rel {abs(ltf-rl)/rl:.2e}  ({time.time()-t0:.0f}s)", flush=True)
