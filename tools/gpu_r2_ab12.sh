timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in base pv; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/graph_step.py --steps 300 > gpurun_out/ab12_graph_$v.jsonl 2>/dev/null; python3 -c "
import json
for l in open('gpurun_out/ab12_graph_$v.jsonl'):
    d=json.loads(l); print('$v', d['config'],d['optimizer'],d['mode'],'ms',round(d['ms'],4),'Gp/s',round(d['gparams_per_s'],1))
"; done
VARIANTS="base:build/base/lib.so: pv:build/pv/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -4
