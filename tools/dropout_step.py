"""One Transformer-base update at dropout 0.1 (device Philox masks) after
warm-up, for ncu captures of the dropout kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_00344_b200 import CONFIGS, TOKEN_BUDGET, config_text, mtk as M

cfg = config_text(**dict(CONFIGS["base"], dropout=0.1))
model = M.Model(cfg)
g = M.ExpressionGraph(1)
model.register_params(g)
g.clear()
adam = M.Adam(M.adam_defaults_for(cfg))
avg = M.AveragedParameters(0.9999)
opts = M.TrainOptions()
opts.token_budget = TOKEN_BUDGET["base"]
st = M.SyncStepper(model, g, adam, avg, opts)
batches = M.make_batches(M.synth_examples(2000, 32000), TOKEN_BUDGET["base"], 1, True)
for i in range(3):
    st.update([batches[i]], i, True)
M.sync()
