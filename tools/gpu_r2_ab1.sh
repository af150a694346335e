# K13 split + scaled roots: parity suite on the product build, then A/B of
# the variants under the power cap.
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab1_tests.txt 2>&1; tail -3 gpurun_out/ab1_tests.txt
STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab1.txt
