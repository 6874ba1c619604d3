# RNN scan iteration: persistent-scan parity tests, then phase profile and bench of shallow/deep
python -m pytest tests/test_rnn_persist_gpu.py tests/test_parity_fullsize_gpu.py -x -q -k "shallow or deep or persist" > gpurun_out/rnn_tests.log 2>&1; echo rc=$? >> gpurun_out/rnn_tests.log
for c in shallow deep; do MTK_RNN_PROF=1 timeout 300 python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/prof_$c.json 2> gpurun_out/prof_$c.err; done
for c in shallow deep; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2>&1; done
