FO_LIB_PATH=$PWD/build/mq/lib.so timeout 900 python -m pytest tests/test_gpu_primitives.py -q -k "rcp_approx or momentum_preimage" 2>&1 | tail -2
FO_LIB_PATH=$PWD/build/mq/lib.so timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FO_LIB_PATH=$PWD/build/mq/lib.so timeout 400 python tools/parity_stress.py --seconds 240 --seed 31 --layouts 2>&1 | tail -1
VARIANTS="base:build/base/lib.so: mq:build/mq/lib.so:" STEPS=150 REPS=3 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab11.txt
