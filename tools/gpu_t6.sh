set -x
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_torch_optim.py -x -q -m gpu 2>&1 | tail -5
for k in ${KERNELS:-ws}; do
  FO_KERNEL=$k timeout 300 python bench.py --config llama31_8b --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/b_$k.json 2> gpurun_out/b_$k.err
  python -c "import json;d=json.load(open('gpurun_out/b_$k.json'));print('$k', round(d['value'],1), round(d['roofline']['frac'],3), d['clocks'], 'per-GHz', round(d['value']/d['clocks']['sm_mhz']*1000,1))"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:step_ws -s 3 -c 1 -o gpurun_out/prof_ws -f python bench.py --config gpt2_medium --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_ws.log 2>&1
tail -2 gpurun_out/ncu_ws.log
