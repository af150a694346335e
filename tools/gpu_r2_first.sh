nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/r2a_box.txt
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2a_pytest.txt 2>&1; tail -3 gpurun_out/r2a_pytest.txt
timeout 900 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; tail -2 gpurun_out/r2a_bench.err; cat gpurun_out/r2a_bench.json | head -c 600
