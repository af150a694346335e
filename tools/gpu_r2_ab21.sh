# fix-up kernel as a programmatic launch with the implicit trigger (fx1) vs plain launch (base = in-tree)
mkdir -p build/base && cp paper_2602_23349_b200/libflashoptim_b200.so build/base/lib.so
FO_LIB_PATH=$PWD/build/fx1/lib.so timeout 900 python -m pytest tests/test_gpu_capturable.py tests/test_gpu_pdl.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for rep in 1 2; do for v in base fx1; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/graph_step.py --steps 300 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v', d['config'], d['optimizer'], d['mode'], 'ms', round(d['ms'],4), 'err', d['device_errors'])
"; done; done
CFGS="resnet50:sgd resnet50:lion" VARIANTS="base:build/base/lib.so: fx1:build/fx1/lib.so:" STEPS=40 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tail -8
VARIANTS="base:build/base/lib.so: fx1:build/fx1/lib.so:" STEPS=150 REPS=1 bash tools/gpu_ab_power.sh 2>&1 | tail -2
