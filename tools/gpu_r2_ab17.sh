# PDL for the fused launch only (in-tree, pdlA) vs fused + fix-up (pdl1) vs none (pdl0)
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_driver.py 2>&1 | tail -2
for rep in 1 2; do for v in pdlA pdl1 pdl0; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/graph_step.py --steps 300 > gpurun_out/ab17_graph_$v.jsonl 2>/dev/null; python3 -c "
import json
for l in open('gpurun_out/ab17_graph_$v.jsonl'):
    d=json.loads(l)
    print('$v', d['config'],d['optimizer'],d['mode'],'ms',round(d['ms'],4), 'err', d['device_errors'])
"; done; done
CFGS="resnet50:sgd resnet50:lion gpt2_medium:adamw" VARIANTS="pdlA:build/pdlA/lib.so: pdl1:build/pdl1/lib.so: pdl0:build/pdl0/lib.so:" STEPS=40 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -18
VARIANTS="pdlA:build/pdlA/lib.so: pdl1:build/pdl1/lib.so: pdl0:build/pdl0/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -6
for rep in 1 2; do for v in pdlA pdl0; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/bench_gpt2_train.py --modes flash,flash_release --steps 20 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$v', {k: d[k] for k in d if k in ('mode','ms_per_step','tokens_per_s','opt_ms','optimizer_ms')})
"; done; done
