timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab10_tests.txt 2>&1; tail -1 gpurun_out/ab10_tests.txt
for v in base fx; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/graph_step.py --steps 300 > gpurun_out/ab10_graph_$v.jsonl 2>/dev/null; python3 -c "
import json
for l in open('gpurun_out/ab10_graph_$v.jsonl'):
    d=json.loads(l); print('$v', d['config'],d['optimizer'],d['mode'],'ms',round(d['ms'],4),'Gp/s',round(d['gparams_per_s'],1),'frac',round(d['frac_of_measured_hbm'],3))
"; done
VARIANTS="base:build/base/lib.so: fx:build/fx/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab10.txt
