MTK_PKG_ROOT=$PWD/ab64 timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -1
python tools/gemm_bench.py 20 > gpurun_out/gemm_32.txt 2>&1
MTK_PKG_ROOT=$PWD/ab64 python tools/gemm_bench.py 20 > gpurun_out/gemm_64.txt 2>&1
for i in 1 2; do
python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bk32', d['value'], d['ms_per_step'])"
MTK_PKG_ROOT=$PWD/ab64 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bk64', d['value'], d['ms_per_step'])"
done
