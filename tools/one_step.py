"""Warm-up updates then ONE timed update of a config (for ncu launch lists):
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/one_step.py base 3
The last update's kernels are the ones after the marker kernel (mtkc_gpu_sleep)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_00344_b200 import CONFIGS, TOKEN_BUDGET, config_text, mtk as M

name = sys.argv[1] if len(sys.argv) > 1 else "base"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = config_text(**CONFIGS[name])
model = M.Model(cfg)
g = M.ExpressionGraph(1)
model.register_params(g)
g.clear()
adam = M.Adam(M.adam_defaults_for(cfg))
avg = M.AveragedParameters(0.9999)
opts = M.TrainOptions()
opts.token_budget = TOKEN_BUDGET[name]
st = M.SyncStepper(model, g, adam, avg, opts)
batches = M.make_batches(M.synth_examples(2000, CONFIGS[name]["vocab"]), TOKEN_BUDGET[name], 1, True)
for i in range(warm):
    st.update([batches[i]], i, True)
M.sync()
M.gpu_sleep(1000)  # marker kernel
st.update([batches[warm]], warm, True)
M.sync()
