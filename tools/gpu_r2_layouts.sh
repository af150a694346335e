# fused-kernel optional layouts: parity + throughput
timeout 1200 python -m pytest tests/test_gpu_layouts.py tests/test_gpu_g32.py tests/test_gpu_parity.py tests/test_gpu_torch_optim.py -x -q > gpurun_out/lay_tests.txt 2>&1; tail -3 gpurun_out/lay_tests.txt
timeout 600 python tools/bench_variants.py --config gpt2_medium > gpurun_out/lay_var_gpt2.jsonl 2>&1; cat gpurun_out/lay_var_gpt2.jsonl | cut -c1-300
FO_FAST_LAYOUTS=0 timeout 600 python tools/bench_variants.py --config gpt2_medium > gpurun_out/lay_var_gpt2_g32.jsonl 2>&1; cat gpurun_out/lay_var_gpt2_g32.jsonl | cut -c1-300
timeout 900 python tools/bench_variants.py --config llama31_8b --steps 5 > gpurun_out/lay_var_llama.jsonl 2>&1; cat gpurun_out/lay_var_llama.jsonl | cut -c1-300
