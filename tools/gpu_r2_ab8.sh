VARIANTS="ws:paper_2602_23349_b200/libflashoptim_b200.so: ldg:paper_2602_23349_b200/libflashoptim_b200.so:FO_KERNEL=mt" STEPS=150 REPS=2 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab8.txt
