FO_LIB_PATH=$PWD/build/e_ncw16/lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lists.py -x -q > gpurun_out/ab2_tests.txt 2>&1; tail -2 gpurun_out/ab2_tests.txt
VARIANTS="b_new e_ncw16" bash tools/gpu_r2_ncu_ab.sh 2>&1 | python3 -c "
import sys,ast
for l in sys.stdin:
    v,d=l.split(' ',1); d=ast.literal_eval(d); t=d['gpu__time_duration.sum']; print(v, 'ms', round(sum(t)/len(t)/1e6,3), 'inst', d['smsp__inst_executed.sum'][0], 'issue', d['smsp__issue_active.avg.pct_of_peak_sustained_active'][0])
"
VARIANTS="b:build/b_new/lib.so: e:build/e_ncw16/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab2.txt
