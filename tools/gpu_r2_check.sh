# Round-2 re-entry check: full GPU suite, smoke, default bench.
set -x
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/chk_box.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/chk_tests.txt 2>&1; tail -5 gpurun_out/chk_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk_smoke.txt 2>&1; tail -2 gpurun_out/chk_smoke.txt
timeout 900 python bench.py > gpurun_out/chk_bench.json 2> gpurun_out/chk_bench.err; tail -3 gpurun_out/chk_bench.err
