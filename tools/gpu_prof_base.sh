set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py --config llama31_8b --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_base.json 2> gpurun_out/b_base.err
cat gpurun_out/b_base.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_tma -s 3 -c 1 -o gpurun_out/prof_base -f python bench.py --config gpt2_medium --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_base.log 2>&1
tail -5 gpurun_out/ncu_base.log
