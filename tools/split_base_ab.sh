for r in 1 2; do for ms in 4 6 8 12; do MTK_GEMM_MAXSPLIT=$ms python bench.py --no-cpu-baseline > gpurun_out/splitb_${ms}_$r.json 2>/dev/null; done; done
