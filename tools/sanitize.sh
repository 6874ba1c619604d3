#!/bin/bash
# compute-sanitizer runs over small parity cases (memcheck: out-of-bounds /
# misaligned accesses; racecheck: shared-memory hazards)
O=gpurun_out/sanitizer
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name tool pytest-args...
  local name=$1 tool=$2; shift 2
  timeout 900 $CS --tool $tool --print-limit 20 python -m pytest -x -q -p no:cacheprovider "$@" > $O/$name.log 2>&1
  echo "$name ($tool): rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $O/$name.log | tr '\n' ' ')"
}
run gemm memcheck tests/test_gemm_gpu.py
run ops memcheck tests/test_ops_gpu.py -k "layernorm or attention or cross_entropy or embed"
run rnn_persist memcheck "tests/test_rnn_persist_gpu.py::test_persistent_scan_matches_per_step_path[shallow-d256]"
run dropout memcheck tests/test_dropout_gpu.py -k device
run lstm memcheck tests/test_lstm_gpu.py
run attn_race racecheck tests/test_ops_gpu.py -k "attention_tensor_core"
run ln_race racecheck tests/test_ops_gpu.py -k "layernorm"
