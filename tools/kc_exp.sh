for kc in 2 4 8; do export MTK_RNN_KCH=$kc; timeout 300 python bench.py --config deep --no-cpu-baseline --steps 10 --warmup 3 > /tmp/b.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/b.json'));print('KCH', $kc, d['value'])"; done
unset MTK_RNN_KCH
for kc in 4 8 12 16; do export MTK_RNN_KCB=$kc; timeout 300 python bench.py --config deep --no-cpu-baseline --steps 10 --warmup 3 > /tmp/b.json 2>/dev/null; python -c "import json;d=json.load(open('/tmp/b.json'));print('KCB', $kc, d['value'])"; done
