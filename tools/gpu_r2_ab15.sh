# fix-up in the fused kernel (FO_INLINE_FIX=1, in-tree) vs the separate fix-up launch (build/ifx0)
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_driver.py 2>&1 | tail -3
for rep in 1 2; do for v in ifx1 ifx0; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/graph_step.py --steps 300 > gpurun_out/ab15_graph_$v.jsonl 2>/dev/null; python3 -c "
import json
for l in open('gpurun_out/ab15_graph_$v.jsonl'):
    d=json.loads(l)
    print('$v', d['config'],d['optimizer'],d['mode'],'ms',round(d['ms'],4))
"; done; done
CFGS="resnet50:sgd resnet50:lion gpt2_medium:adamw" VARIANTS="ifx1:build/ifx1/lib.so: ifx0:build/ifx0/lib.so:" STEPS=40 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -12
VARIANTS="ifx1:build/ifx1/lib.so: ifx0:build/ifx0/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -4
