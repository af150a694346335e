FO_LIB_PATH=$PWD/build/g_ws2_16/lib.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lists.py -x -q > gpurun_out/ab4_tests.txt 2>&1; tail -2 gpurun_out/ab4_tests.txt
VARIANTS="g16:build/g_ws2_16/lib.so: e16:build/e_ncw16/lib.so:" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab4.txt
