O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 2 -c 1 -o $O/r02b_gemm_logits_pair -f python tools/gemm_one.py 6500 32000 512 0 1 > $O/ncu_g1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 2 -c 1 -o $O/r02b_gemm_ffn1_pair -f python tools/gemm_one.py 6500 2048 512 0 0 > $O/ncu_g2.log 2>&1
MTK_GEMM_NO_PAIR=1 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 2 -c 1 -o $O/r02b_gemm_ffn1_single -f python tools/gemm_one.py 6500 2048 512 0 0 > $O/ncu_g3.log 2>&1
python tools/ncu_summary.py $O/r02b_gemm_logits_pair.ncu-rep $O/r02b_gemm_ffn1_pair.ncu-rep $O/r02b_gemm_ffn1_single.ncu-rep $O/r02b_xent.ncu-rep > $O/r02b_ncu_summary.txt 2>&1
for f in r02b_gemm_logits_pair r02b_gemm_ffn1_pair r02b_gemm_ffn1_single; do
  ncu -i $O/$f.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed > $O/$f.raw.csv 2>&1
done
