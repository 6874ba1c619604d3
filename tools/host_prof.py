"""Host-side cost of one Transformer-base update: graph build / forward
(launch) / backward (launch) milliseconds, and the host cost of one
mtkc_gemm call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1804_00344_b200 import CONFIGS, TOKEN_BUDGET, cabi, config_text, mtk as M

cfg = config_text(**CONFIGS["base"])
model = M.Model(cfg)
g = M.ExpressionGraph(1)
model.register_params(g)
g.clear()
adam = M.Adam(M.adam_defaults_for(cfg))
avg = M.AveragedParameters()
opts = M.TrainOptions()
opts.token_budget = TOKEN_BUDGET["base"]
st = M.SyncStepper(model, g, adam, avg, opts)
batches = M.make_batches(M.synth_examples(4000, 32000), 16384, 1, True)
for i in range(3):
    st.update([batches[i]], i, True)
h0 = st.host_times()
M.sync()
M.gpu_sleep(2_000_000)
t0 = time.perf_counter()
n = 5
for i in range(3, 3 + n):
    st.update([batches[i]], i, False)
t1 = time.perf_counter()
h1 = st.host_times()
print("host ms/step total %.2f  build %.2f  forward %.2f  backward %.2f" % (
    (t1 - t0) * 1e3 / n, (h1[0] - h0[0]) / n, (h1[1] - h0[1]) / n, (h1[2] - h0[2]) / n))
M.sync()

# unthrottled host cost: launch queue empty at the start of every step
hs = []
for i in range(8, 14):
    M.sync()
    h0 = st.host_times()
    t0 = time.perf_counter()
    st.update([batches[i]], i, False)
    t1 = time.perf_counter()
    h1 = st.host_times()
    hs.append(((t1 - t0) * 1e3, h1[0] - h0[0], h1[1] - h0[1], h1[2] - h0[2]))
M.sync()
for h in hs:
    print("queue-empty step: host %.2f ms (build %.2f fwd %.2f bwd %.2f)" % h)

# host cost of one GEMM call (GPU kept busy so launches do not block)
A = torch.randn(6629, 512, device="cuda")
B = torch.randn(512, 512, device="cuda")
C = torch.empty(6629, 512, device="cuda")
ws = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for prec in (1, 0):
    t0 = time.perf_counter()
    for _ in range(200):
        cabi.gemm(6629, 512, 512, A.data_ptr(), 512, B.data_ptr(), 512, C.data_ptr(), 512,
                  precision=prec, workspace=ws.data_ptr(), workspace_bytes=ws.numel(), stream=s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print("mtkc_gemm host us/call (precision %d): %.1f" % (prec, (t1 - t0) * 1e6 / 200))
