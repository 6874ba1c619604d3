for kc in 2 4 8 16; do export MTK_RNN_KCC=$kc; timeout 300 python bench.py --config shallow --no-cpu-baseline --steps 10 --warmup 3 > /tmp/b.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/b.json'));print('KCC', $kc, d['value'])"; done
unset MTK_RNN_KCC
for kc in 2 4 8 16; do export MTK_RNN_KCX=$kc; timeout 300 python bench.py --config shallow --no-cpu-baseline --steps 10 --warmup 3 > /tmp/b.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/b.json'));print('KCX', $kc, d['value'])"; done
