# programmatic dependent launch of the fused and fix-up kernels (FO_PDL=1, in-tree) vs plain launches (build/pdl0)
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_driver.py 2>&1 | tail -2
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_driver.py 2>&1 | tail -2
for rep in 1 2; do for v in pdl1 pdl0; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/graph_step.py --steps 300 > gpurun_out/ab16_graph_$v.jsonl 2>/dev/null; python3 -c "
import json
for l in open('gpurun_out/ab16_graph_$v.jsonl'):
    d=json.loads(l)
    print('$v', d['config'],d['optimizer'],d['mode'],'ms',round(d['ms'],4), 'err', d['device_errors'])
"; done; done
CFGS="resnet50:sgd resnet50:lion gpt2_medium:adamw" VARIANTS="pdl1:build/pdl1/lib.so: pdl0:build/pdl0/lib.so:" STEPS=40 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -12
VARIANTS="pdl1:build/pdl1/lib.so: pdl0:build/pdl0/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -4
