# bench the in-tree library and any variant libraries under build/*/lib.so
set -x
for lib in paper_2602_23349_b200/libflashoptim_b200.so build/*/lib.so; do
  tag=$(echo $lib | tr '/' '_')
  FO_LIB_PATH=$PWD/$lib python bench.py --config llama31_8b --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bv_$tag.json 2> gpurun_out/bv_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/bv_$tag.json'));print('$lib', round(d['value'],1), round(d['roofline']['frac'],3), d['clocks'])" || tail -3 gpurun_out/bv_$tag.err
done
