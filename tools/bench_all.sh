# bench lines for every BASELINE config (+ fp32 base, base at dropout 0.1)
O=gpurun_out
for c in tiny base big shallow deep; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 5 > $O/r02_bench_$c.json 2> $O/r02_bench_$c.err
done
timeout 400 python bench.py --config base --precision fp32 --no-cpu-baseline --steps 10 --warmup 3 > $O/r02_bench_base_fp32.json 2> $O/r02_bench_base_fp32.err
timeout 400 python bench.py --config base --dropout 0.1 --no-cpu-baseline --steps 20 --warmup 5 > $O/r02_bench_base_dropout01.json 2> $O/r02_bench_base_dropout01.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/r02_bench_reference_base.json 2> $O/r02_bench_reference_base.err
for f in $O/r02_bench_*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', d.get('value'), d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), (d.get('cpu_baseline') or {}).get('value'), d.get('dtype'))"; done
