# round-2 final validation (after the layout kernels): full GPU suite, smoke,
# the base step launch list, bench lines for every config
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/r02e_gputest.log 2>&1; tail -3 $O/r02e_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02e_base_launches.csv python tools/one_step.py base 3 > /dev/null 2>&1
python tools/launches.py $O/r02e_base_launches.csv 30 > $O/r02e_base_launches.txt 2>&1
for c in tiny base big shallow deep; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > $O/r02e_bench_$c.json 2> $O/r02e_bench_$c.err
done
timeout 400 python bench.py --config base --precision fp32 --no-cpu-baseline --steps 10 --warmup 3 > $O/r02e_bench_base_fp32.json 2> $O/r02e_bench_base_fp32.err
timeout 400 python bench.py --config base --dropout 0.1 --no-cpu-baseline --steps 20 --warmup 5 > $O/r02e_bench_base_dropout01.json 2> $O/r02e_bench_base_dropout01.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r02e_bench_reference_base.json 2> $O/r02e_bench_reference_base.err
for f in $O/r02e_bench_*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d.get('dtype'))"; done
python tools/gaps.py shallow 3 > $O/r02e_gaps_shallow.txt 2>&1; python tools/gaps.py base 3 > $O/r02e_gaps_base.txt 2>&1
