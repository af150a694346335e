#!/bin/bash
# A/B of build/*/lib.so over several configs, alternating twice on one box:
#   CFGS="llama31_8b:adamw gpt2_medium:adamw resnet50:sgd" ./tools/gpu_ab_cfg.sh
CFGS=${CFGS:-"llama31_8b:adamw llama31_8b:sgd llama31_8b:lion gpt2_medium:adamw resnet50:sgd"}
for cfg in $CFGS; do
  c=${cfg%%:*}; o=${cfg##*:}
  for rep in 1 2; do
    for lib in build/*/lib.so; do
      FO_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config $c --optimizer $o --steps 30 --warmup 5 --no-e2e --no-cpu > gpurun_out/abc.json 2> gpurun_out/abc.err
      python -c "import json;d=json.load(open('gpurun_out/abc.json'));c=d['clocks'];print('$c $o $lib', round(d['value'],1), c['sm_mhz'], 'per-GHz', round(d['value']/c['sm_mhz']*1000,1))" || tail -3 gpurun_out/abc.err
    done
  done
done
