# alternate variant libraries A/B/... twice on the same box (per-GHz comparison)
OPT=${OPT:-adamw}
for rep in 1 2; do
for lib in build/*/lib.so; do
  tag=$(echo $lib | tr '/' '_')
  FO_LIB_PATH=$PWD/$lib timeout 300 python bench.py --optimizer $OPT --steps 40 --warmup 5 --no-e2e --no-cpu > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$tag.json'));c=d['clocks'];print('$lib', round(d['value'],1), c['sm_mhz'], c['power_w'], 'per-GHz', round(d['value']/c['sm_mhz']*1000,1))" || tail -3 gpurun_out/ab_$tag.err
done
done
