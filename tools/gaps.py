"""Idle device time between consecutive kernels/copies of plain training
updates (CUPTI records via torch.profiler): total busy vs wall, and the
largest gaps by (previous, next) activity.

  python tools/gaps.py [config] [steps]
"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch.profiler as tp

from paper_1804_00344_b200 import CONFIGS, TOKEN_BUDGET, config_text, mtk as M

name = sys.argv[1] if len(sys.argv) > 1 else "base"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
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
for i in range(6):
    st.update([batches[i]], i, True)
M.sync()
M.gpu_sleep(3_000_000)  # the host queues the profiled updates behind a sleep
with tp.profile(activities=[tp.ProfilerActivity.CUDA]) as prof:
    for i in range(6, 6 + steps):
        st.update([batches[i]], i, False)
    M.sync()
ev = []
for e in prof.events():
    if "CUDA" not in str(getattr(e, "device_type", "")):
        continue
    ev.append((e.time_range.start, e.time_range.end, e.name[:160]))
ev.sort()
ev = [x for x in ev if "sleep" not in x[2]]
t0, t1 = ev[0][0], max(x[1] for x in ev)
busy, prev_end, prev_name = 0.0, None, None
gaps = collections.defaultdict(lambda: [0, 0.0])
kinds = collections.Counter()
for s, e, n in ev:
    kinds[n.split("<")[0].split("(")[0][:40]] += 1
    if prev_end is not None and s > prev_end:
        k = (prev_name.split("<")[0][:38], n.split("<")[0][:38])
        gaps[k][0] += 1
        gaps[k][1] += s - prev_end
    busy += e - (s if prev_end is None else max(s, prev_end)) if prev_end is None or e > prev_end else 0
    if prev_end is None or e > prev_end:
        prev_end, prev_name = e, n
wall = (t1 - t0) / steps
print(f"{name}: wall {wall/1e3:.3f} ms/update, busy {busy/steps/1e3:.3f} ms, idle {(wall - busy/steps)/1e3:.3f} ms")
for k, (c, us) in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{us/steps:9.1f} us/update {c/steps:6.1f}x  {k[0]} -> {k[1]}")
print("non-kernel activities:", {k: v for k, v in kinds.items() if "emcpy" in k or "emset" in k})
# exclusive device time per activity name (each instant to the activity that finishes it)
per = collections.defaultdict(lambda: [0, 0.0])
pe = None
for s_, e_, n in ev:
    ex = e_ - (s_ if pe is None else max(s_, pe))
    pe = e_ if pe is None else max(pe, e_)
    k = n.replace("(anonymous namespace)::", "").replace("mtkc::", "")
    k = k.split("(")[0].split("<")[0][:60]
    per[k][0] += 1
    per[k][1] += max(ex, 0.0)
print("exclusive time per activity (us/update, launches/update):")
for k, (c, us) in sorted(per.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{us/steps:9.1f} {c/steps:6.1f}x  {k}")
