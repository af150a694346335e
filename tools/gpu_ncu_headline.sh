# ncu on the HEADLINE configuration (Llama-3.1-8B list, 8.03 G params):
# 1) launch list of the bench command (time only, cold/serialised)
# 2) one --set full capture of the fused step (kernel replay, memory saved/restored by ncu)
# 3) the same on ResNet-50 SGD and GPT-2-medium AdamW
set -x
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_llama8b.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_launches.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:step_ws -s 3 -c 1 -o gpurun_out/ncu_full_llama8b -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_full_llama8b.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ws -s 3 -c 1 -o gpurun_out/ncu_full_resnet_sgd -f python bench.py --config resnet50 --optimizer sgd --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_full_resnet.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ws -s 3 -c 1 -o gpurun_out/ncu_full_gpt2 -f python bench.py --config gpt2_medium --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > gpurun_out/ncu_full_gpt2.log 2>&1
ls -la gpurun_out/*.ncu-rep
