for ms in 1 2 4 8; do for c in shallow deep; do MTK_GEMM_MAXSPLIT=$ms python bench.py --config $c --no-cpu-baseline > gpurun_out/split_${c}_$ms.json 2>/dev/null; done; done
