# parity on the default kernel, then bench the in-tree library (each FO_KERNEL in $KERNELS)
# and any variant libraries under build/*/lib.so
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -x -q -m gpu 2>&1 | tail -3
for k in ${KERNELS:-ws}; do
  FO_KERNEL=$k timeout 300 python bench.py --config llama31_8b --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/bk_$k.json 2> gpurun_out/bk_$k.err
  python -c "import json;d=json.load(open('gpurun_out/bk_$k.json'));print('kernel $k', round(d['value'],1), round(d['roofline']['frac'],3), d['clocks'], 'per-GHz', round(d['value']/d['clocks']['sm_mhz']*1000,1))" || tail -3 gpurun_out/bk_$k.err
done
for lib in build/*/lib.so; do
  [ -f "$lib" ] || continue
  tag=$(echo $lib | tr '/' '_')
  FO_LIB_PATH=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
  FO_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config llama31_8b --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/bv_$tag.json 2> gpurun_out/bv_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/bv_$tag.json'));print('$lib', round(d['value'],1), round(d['roofline']['frac'],3), d['clocks'], 'per-GHz', round(d['value']/d['clocks']['sm_mhz']*1000,1))" || tail -3 gpurun_out/bv_$tag.err
done
