for v in rc rcn nar; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lists.py -x -q > gpurun_out/ab5_tests_$v.txt 2>&1; echo $v; tail -1 gpurun_out/ab5_tests_$v.txt; done
VARIANTS="base:build/base/lib.so: rc:build/rc/lib.so: rcn:build/rcn/lib.so: nar:build/nar/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab5.txt
VARIANTS="base rc rcn nar" bash tools/gpu_r2_ncu_ab.sh 2>&1 | python3 -c "
import sys,ast
for l in sys.stdin:
    try:
        v,d=l.split(' ',1); d=ast.literal_eval(d); t=d['gpu__time_duration.sum']; print(v, 'ms', round(sum(t)/len(t)/1e6,3), 'inst', d['smsp__inst_executed.sum'][0], 'issue', d['smsp__issue_active.avg.pct_of_peak_sustained_active'][0])
    except Exception as e: print(l[:200])
"
