# Round-2 artifacts on the final kernel: headline bench (defaults), reference
# arm, other configs, t0=10, ncu launch list of the headline command and a
# --set full capture (with source) of the headline launch, GPU tests.
set -x
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/art2_box.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/art2_tests.txt 2>&1; tail -2 gpurun_out/art2_tests.txt
timeout 900 python bench.py > gpurun_out/art2_bench.json 2> gpurun_out/art2_bench.err; tail -2 gpurun_out/art2_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/art2_ref.json 2> gpurun_out/art2_ref.err
for c in "resnet50 sgd" "resnet50 lion" "gpt2_medium adamw" "llama31_8b sgd" "llama31_8b lion"; do
  set -- $c; timeout 300 python bench.py --config $1 --optimizer $2 --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/art2_$1_$2.json 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --t0 10 > gpurun_out/art2_t10.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/art2_launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/art2_launches.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:step_ws -s 3 -c 1 -o gpurun_out/art2_full -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/art2_full.log 2>&1
bash tools/ncu_summary.sh gpurun_out/art2_full.ncu-rep > gpurun_out/art2_full_summary.txt
ncu -i gpurun_out/art2_full.ncu-rep --page source --csv --print-source sass > gpurun_out/art2_sass.csv 2>/dev/null
ncu -i gpurun_out/art2_full.ncu-rep --page details --csv > gpurun_out/art2_details.csv 2>/dev/null
python tools/sass_hist.py gpurun_out/art2_sass.csv 8030261248 > gpurun_out/art2_sass_hist.txt
gzip -f gpurun_out/art2_sass.csv; rm -f gpurun_out/art2_full.ncu-rep
timeout 600 ncu --set full --clock-control none -k regex:step_ws -s 3 -c 1 -o gpurun_out/art2_resnet -f python bench.py --config resnet50 --optimizer sgd --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/art2_resnet.log 2>&1
bash tools/ncu_summary.sh gpurun_out/art2_resnet.ncu-rep > gpurun_out/art2_resnet_summary.txt; rm -f gpurun_out/art2_resnet.ncu-rep
timeout 600 python tools/bench_gpt2_train.py > gpurun_out/art2_gpt2_train.jsonl 2> gpurun_out/art2_gpt2_train.err
