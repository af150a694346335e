timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab3_tests.txt 2>&1; tail -3 gpurun_out/ab3_tests.txt
for v in ws2 ws1; do
  FO_KERNEL=$v timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ncuab3_$v.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncuab3_$v.log 2>&1
  python3 - $v <<'PY'
import csv, sys
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/ncuab3_{v}.csv")) if len(r) > 10]
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
agg = {}
for r in rows[1:]:
    if "step_ws" not in r[ix["Kernel Name"]]: continue
    agg.setdefault(r[ix["Metric Name"]], []).append(float(r[ix["Metric Value"]].replace(",", "")))
t = agg.get("gpu__time_duration.sum", [0])
print(v, "ms", round(sum(t) / len(t) / 1e6, 3), {k: vals[0] for k, vals in agg.items()})
PY
done
VARIANTS="ws2:paper_2602_23349_b200/libflashoptim_b200.so: ws1:paper_2602_23349_b200/libflashoptim_b200.so:FO_KERNEL=ws1 e16:build/e_ncw16/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab3.txt
