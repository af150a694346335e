# A/B: parity tests on the default kernel, then bench each kernel variant
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q -m gpu 2>&1 | tail -5
for k in ${KERNELS:-ws tma}; do
  FO_KERNEL=$k python bench.py --config llama31_8b --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_$k.json 2> gpurun_out/b_$k.err
  python -c "import json;d=json.load(open('gpurun_out/b_$k.json'));print('$k', round(d['value'],1), round(d['roofline']['frac'],3), d['clocks'])"
done
