#!/bin/bash
# round-2 ncu captures (one launch each, --set full) + summaries
set -x
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:rnn_scan_fwd_kernel -c 1 -o $O/r02_rnn_fwd -f python tools/one_step.py shallow 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rnn_scan_bwd_kernel -c 1 -o $O/r02_rnn_bwd -f python tools/one_step.py shallow 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_tc_fwd_kernel -s 20 -c 1 -o $O/r02_attn_fwd -f python tools/one_step.py base 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_tc_bwd_kernel -s 20 -c 1 -o $O/r02_attn_bwd -f python tools/one_step.py base 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:dropout -s 40 -c 2 -o $O/r02_dropout -f python tools/dropout_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:splitk_reduce -s 40 -c 1 -o $O/r02_splitk -f python tools/one_step.py base 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ln_fwd4 -s 40 -c 1 -o $O/r02_lnfwd -f python tools/one_step.py base 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:embed4 -s 2 -c 1 -o $O/r02_embed -f python tools/one_step.py base 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:scatter -s 2 -c 1 -o $O/r02_scatter -f python tools/one_step.py base 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/r02_*.ncu-rep > $O/r02_ncu_summary.txt 2>&1
ls -la $O/*.ncu-rep
