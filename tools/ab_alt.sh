# same-box A/B of the current build against a copy of the previous build in alt_old/
for r in 1 2; do for c in shallow deep; do
  (cd alt_old && python bench.py --config $c --no-cpu-baseline > ../gpurun_out/alt_old_${c}_$r.json 2>/dev/null)
  python bench.py --config $c --no-cpu-baseline > gpurun_out/alt_new_${c}_$r.json 2>/dev/null
done; done
