# round 2: new bench (parity windows, fast-path share, NVML power), ZeRO path (gloo test mode), reference arm
timeout 900 python -m pytest tests/test_gpu_zero2.py -q -x > gpurun_out/r2c_zero2.txt 2>&1; tail -3 gpurun_out/r2c_zero2.txt
( time timeout 900 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err ) 2> gpurun_out/r2c_bench.time; tail -3 gpurun_out/r2c_bench.err; cat gpurun_out/r2c_bench.time
FO_BENCH_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config gpt2_medium --steps 5 --warmup 3 --no-e2e > gpurun_out/r2c_zero_gloo.json 2> gpurun_out/r2c_zero_gloo.err; tail -3 gpurun_out/r2c_zero_gloo.err
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2c_ref.json 2> gpurun_out/r2c_ref.err ) 2> gpurun_out/r2c_ref.time; tail -3 gpurun_out/r2c_ref.err; cat gpurun_out/r2c_ref.time
nproc > gpurun_out/r2c_nproc.txt; free -g >> gpurun_out/r2c_nproc.txt
