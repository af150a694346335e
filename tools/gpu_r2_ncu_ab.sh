# Uncapped per-launch comparison of library variants (ncu serialises launches,
# so the 1000 W cap does not pull the clock) + a full source-level capture of
# the product build on the headline list.
for v in ${VARIANTS:-a_base b_new}; do
  FO_LIB_PATH=$PWD/build/$v/lib.so timeout 900 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ncuab_$v.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncuab_$v.log 2>&1
  python - $v <<'PY'
import csv, sys
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/ncuab_{v}.csv")) if len(r) > 10]
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
agg = {}
for r in rows[1:]:
    if "step_ws" not in r[ix["Kernel Name"]]: continue
    agg.setdefault(r[ix["Metric Name"]], []).append(float(r[ix["Metric Value"]].replace(",", "")))
print(v, {k: [round(x, 3) for x in vals] for k, vals in agg.items()})
PY
done
if [ -n "$FULL" ]; then
  FO_LIB_PATH=$PWD/build/$FULL/lib.so timeout 1800 ncu --set full --clock-control none --import-source on -k regex:step_ws -s 3 -c 1 -o gpurun_out/ncu_full_$FULL -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_full_$FULL.log 2>&1
  bash tools/ncu_summary.sh gpurun_out/ncu_full_$FULL.ncu-rep > gpurun_out/ncu_full_${FULL}_summary.txt
  ncu -i gpurun_out/ncu_full_$FULL.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_$FULL.csv 2>/dev/null
  ncu -i gpurun_out/ncu_full_$FULL.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$FULL.csv 2>/dev/null
  gzip -f gpurun_out/ncu_sass_$FULL.csv
  rm -f gpurun_out/ncu_full_$FULL.ncu-rep
fi
