# bench (no parity) the in-tree library and variant libraries under build/*/lib.so
for lib in paper_2602_23349_b200/libflashoptim_b200.so build/*/lib.so; do
  [ -f "$lib" ] || continue
  tag=$(echo $lib | tr '/' '_')
  FO_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config llama31_8b --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/bo_$tag.json 2> gpurun_out/bo_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/bo_$tag.json'));print('$lib', round(d['value'],1), round(d['roofline']['frac'],3), d['clocks'], 'per-GHz', round(d['value']/d['clocks']['sm_mhz']*1000,1))" || tail -3 gpurun_out/bo_$tag.err
done
