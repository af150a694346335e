# round 2: gpu tests (release/oracle, zero), gpt2 training memory, sanitizers, timeline
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2d_pytest.txt 2>&1; tail -3 gpurun_out/r2d_pytest.txt
timeout 900 python tools/bench_gpt2_train.py > gpurun_out/r2d_gpt2_train.jsonl 2> gpurun_out/r2d_gpt2_train.err; echo "train rc=$?"; tail -2 gpurun_out/r2d_gpt2_train.err
timeout 900 python tools/bench_gpt2_train.py --batch 1 --seq 128 --checkpointing --steps 10 --warmup 3 > gpurun_out/r2d_gpt2_train_small.jsonl 2> gpurun_out/r2d_gpt2_train_small.err; echo "small rc=$?"; tail -2 gpurun_out/r2d_gpt2_train_small.err
timeout 900 python tools/timeline.py --out gpurun_out/timeline > gpurun_out/r2d_timeline.txt 2>&1; echo "timeline rc=$?"; tail -2 gpurun_out/r2d_timeline.txt
bash tools/gpu_sanitize.sh
