# final build (fused + fix-up launches programmatic): GPU suite, smoke, memcheck, default bench, small lists
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_driver.py 2>&1 | tail -1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_driver.py 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; tail -1 gpurun_out/f2_bench.err
for c in "resnet50 sgd" "resnet50 lion" "gpt2_medium adamw"; do
  set -- $c; timeout 300 python bench.py --config $1 --optimizer $2 --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/f2_$1_$2.json 2>&1
done
timeout 600 python tools/graph_step.py --steps 300 > gpurun_out/f2_graph.jsonl 2>/dev/null
