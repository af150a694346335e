# the whole GPU test suite, then the config-5 training benchmark
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
timeout 900 python tools/bench_gpt2_train.py > gpurun_out/gpt2_train.jsonl 2> gpurun_out/gpt2_train.err; echo "rc=$?"
cat gpurun_out/gpt2_train.jsonl; tail -3 gpurun_out/gpt2_train.err
