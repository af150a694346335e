# ncu --set full on the fused kernel's optional layouts and on SGD (Llama-8B list)
for v in int16 linear; do
  timeout 900 ncu --set full --clock-control none -k regex:step_ws -s 3 -c 1 -o gpurun_out/ncu_$v -f python tools/bench_variants.py --config llama31_8b --variants $v --steps 2 --warmup 3 > gpurun_out/ncu_$v.log 2>&1
  bash tools/ncu_summary.sh gpurun_out/ncu_$v.ncu-rep > gpurun_out/ncu_${v}_summary.txt; rm -f gpurun_out/ncu_$v.ncu-rep
done
timeout 900 ncu --set full --clock-control none -k regex:step_ws -s 3 -c 1 -o gpurun_out/ncu_sgd -f python bench.py --optimizer sgd --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_sgd.log 2>&1
bash tools/ncu_summary.sh gpurun_out/ncu_sgd.ncu-rep > gpurun_out/ncu_sgd_summary.txt; rm -f gpurun_out/ncu_sgd.ncu-rep
head -4 gpurun_out/ncu_int16_summary.txt gpurun_out/ncu_linear_summary.txt gpurun_out/ncu_sgd_summary.txt
