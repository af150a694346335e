timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do for v in ei1 ei0; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/graph_step.py --steps 300 > gpurun_out/ab14_graph_$v.jsonl 2>/dev/null; python3 -c "
import json
for l in open('gpurun_out/ab14_graph_$v.jsonl'):
    d=json.loads(l)
    if d['mode']=='launch': print('$v', d['config'],d['optimizer'],'ms',round(d['ms'],4))
"; done; done
VARIANTS="ei1:build/ei1/lib.so: ei0:build/ei0/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -4
