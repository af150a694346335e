for v in er cw1; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1; done
VARIANTS="base:build/base/lib.so: er:build/er/lib.so: cw1:build/cw1/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab9.txt
