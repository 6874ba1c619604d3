"""Per-kernel-class HBM traffic of one training update from an ncu CSV with
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(the kernels after the last gpu_sleep marker, tools/one_step.py).  Writes the
JSON that bench.py reports as roofline.traffic (bytes per launch)."""
import collections
import csv
import json
import sys

CLASSES = [("gemm_tf32_tc_kernel", "gemm_tc"), ("attn_tc", "attention"), ("attn_", "attention"),
           ("ln_", "layernorm"), ("colred_final", "layernorm"), ("colsum", "colsum"),
           ("xent", "xent"), ("adam_ema", "adam_ema"), ("splitk_reduce", "gemm_tc")]

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, vi, ui = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
idi = h.index('ID')
launches = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    rec = launches.setdefault(r[idi], {"name": r[ki]})
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    if r[mi] == 'gpu__time_duration.sum':
        v = v / 1e3 if u in ('nsecond', 'ns') else (v if u in ('usecond', 'us') else v * 1e3)
        rec['us'] = v
    else:
        scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}.get(u, 1)
        rec[r[mi]] = v * scale
recs = list(launches.values())
last = max(i for i, r in enumerate(recs) if 'sleep' in r['name'])
agg = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
for r in recs[last + 1:]:
    cls = next((c for pat, c in CLASSES if pat in r['name']), "other")
    a = agg[cls]
    a["launches"] += 1
    a["us"] += r.get('us', 0.0)
    a["dram_bytes"] += r.get('dram__bytes_read.sum', 0.0) + r.get('dram__bytes_write.sum', 0.0)
out = {k: dict(v, dram_bytes_per_launch=v["dram_bytes"] / max(v["launches"], 1)) for k, v in agg.items()}
json.dump({"source": sys.argv[1], "classes": out}, open(sys.argv[2], "w"), indent=1)
for k, v in sorted(out.items(), key=lambda x: -x[1]["us"]):
    print(f"{k:12s} {v['launches']:4d} launches {v['us']/1e3:7.3f} ms  {v['dram_bytes']/1e9:7.3f} GB  "
          f"{v['dram_bytes']/max(v['us'],1e-9)/1e3:7.1f} GB/s")
