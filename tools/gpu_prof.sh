# ncu full capture of the fused step on GPT-2-medium shapes (354.8M params)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ws -s 3 -c 1 -o gpurun_out/prof_ws -f python bench.py --config gpt2_medium --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_ws.log 2>&1
tail -2 gpurun_out/ncu_ws.log
