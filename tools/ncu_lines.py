"""Aggregate ncu source-page (cuda,sass) stall samples per CUDA source line.
usage: ncu -i rep --page source --csv --print-source cuda,sass ... > x.csv; python tools/ncu_lines.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] not in ("", "Line No", "Function Name") and len(r) > 6:
        try:
            out.append((int(r[4]), int(r[6]) if r[6].isdigit() else 0, f, r[0], r[1][:100]))
        except ValueError:
            pass
tot = sum(o[0] for o in out)
print("total samples", tot)
for o in sorted(out, reverse=True)[:n]:
    print(f"{o[0]:7d} {100*o[0]/tot:5.1f}% {o[2]}:{o[3]}  {o[4]}")
