"""Per-call-shape device-time breakdown of one training update
(mtkc_prof_enable(2)); prints classes sorted by time.

  python tools/step_prof.py [config] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_00344_b200 import CONFIGS, TOKEN_BUDGET, config_text, mtk as M

name = sys.argv[1] if len(sys.argv) > 1 else "base"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = config_text(**CONFIGS[name])
M.set_precision("tf32")
model = M.Model(cfg)
g = M.ExpressionGraph(1)
model.register_params(g)
g.clear()
adam = M.Adam(M.adam_defaults_for(cfg))
avg = M.AveragedParameters(0.9999)
opts = M.TrainOptions()
opts.token_budget = TOKEN_BUDGET[name]
st = M.SyncStepper(model, g, adam, avg, opts)
batches = M.make_batches(M.synth_examples(3000, CONFIGS[name]["vocab"]), TOKEN_BUDGET[name], 1, True)
for i in range(4):
    st.update([batches[i]], i, True)
M.sync()
M.gpu_sleep(1_500_000)
M.prof_enable(2)
e0 = M.event_record()
for i in range(4, 4 + steps):
    st.update([batches[i]], i, True)
e1 = M.event_record()
step_ms = M.event_elapsed_ms(e0, e1) / steps
rep = M.prof_report()
M.prof_enable(0)
rows = []
for line in rep.strip().splitlines():
    k, n, ms, work = line.split()
    rows.append((float(ms) / steps, int(n) / steps, float(work) / steps, k))
rows.sort(reverse=True)
tot = sum(r[0] for r in rows)
print(f"step {step_ms:.3f} ms (events around calls; profiled sum {tot:.3f} ms)")
for ms, n, work, k in rows:
    per = ms / max(n, 1)
    rate = work / (ms / 1e3) if ms > 0 else 0
    unit = "TFLOP/s" if k.startswith(("gemm", "attention")) else "GB/s"
    rate = rate / 1e12 if unit == "TFLOP/s" else rate / 1e9
    print(f"{ms:8.3f} ms {100 * ms / step_ms:5.1f}% {n:6.1f}x {per * 1e3:8.1f} us {rate:8.1f} {unit:7s} {k}")
