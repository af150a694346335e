# Round artifacts: headline bench (defaults), reference arm, other configs,
# ncu launch list of the headline command and a full capture on GPT-2 shapes.
set -x
timeout 900 python bench.py > gpurun_out/art_bench.json 2> gpurun_out/art_bench.err; tail -2 gpurun_out/art_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/art_ref.json 2> gpurun_out/art_ref.err
timeout 300 python bench.py --config resnet50 --optimizer sgd --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/art_resnet_sgd.json 2>&1
timeout 300 python bench.py --config resnet50 --optimizer lion --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/art_resnet_lion.json 2>&1
timeout 300 python bench.py --config gpt2_medium --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/art_gpt2.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --t0 10 > gpurun_out/art_bench_t10.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/art_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/art_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ws -s 3 -c 1 -o gpurun_out/art_prof -f python bench.py --config gpt2_medium --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/art_prof.log 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/art_box.txt
timeout 300 python bench.py --optimizer sgd --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/art_llama_sgd.json 2>&1
timeout 300 python bench.py --optimizer lion --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/art_llama_lion.json 2>&1
timeout 900 python tools/bench_gpt2_train.py > gpurun_out/art_gpt2_train.jsonl 2> gpurun_out/art_gpt2_train.err
timeout 300 python tools/bench_variants.py --config gpt2_medium > gpurun_out/art_variants.jsonl 2>&1
