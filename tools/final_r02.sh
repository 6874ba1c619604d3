# round-2 final validation: full GPU suite, smoke, ncu of Adam + fused CE + persistent scan,
# bench lines for every config
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r02_gputest.log 2>&1; tail -3 $O/r02_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
ncu --set full --clock-control none -k regex:adam_ema -c 1 -o $O/r02_adam -f python tools/one_step.py base 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:xent_fused -c 1 -o $O/r02_xent -f python tools/one_step.py base 1 > /dev/null 2>&1
ncu --set full --clock-control none -k regex:rnn_scan_fwd -s 1 -c 1 -o $O/r02_rnn_fwd_dec -f python tools/one_step.py deep 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/r02_adam.ncu-rep $O/r02_xent.ncu-rep $O/r02_rnn_fwd_dec.ncu-rep > $O/r02_ncu_summary2.txt 2>&1
cat $O/r02_ncu_summary2.txt | grep -E "==|duration|dram|tensor"
bash tools/bench_all.sh
