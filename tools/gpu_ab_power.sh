#!/bin/bash
# A/B of library builds and env switches on one box, alternating REPS times,
# with NVML instantaneous power:
#   VARIANTS="base:build/a_base/lib.so: ldg:build/a_base/lib.so:FO_KERNEL=mt" REPS=2 ./tools/gpu_ab_power.sh
# (default: every build/*/lib.so with no extra env)
CFGS=${CFGS:-"llama31_8b:adamw"}
REPS=${REPS:-2}
STEPS=${STEPS:-30}
if [ -z "$VARIANTS" ]; then
  for lib in build/*/lib.so; do VARIANTS="$VARIANTS $(basename $(dirname $lib)):$lib:"; done
fi
for cfg in $CFGS; do
  c=${cfg%%:*}; o=${cfg##*:}
  for rep in $(seq $REPS); do
    for v in $VARIANTS; do
      name=${v%%:*}; rest=${v#*:}; lib=${rest%%:*}; envs=${rest#*:}
      env FO_LIB_PATH=$PWD/$lib ${envs//,/ } timeout 300 python bench.py --config $c --optimizer $o --steps $STEPS --warmup 5 --no-e2e --no-cpu --no-parity $EXTRA > gpurun_out/abp.json 2> gpurun_out/abp.err
      python - "$c" "$o" "$name" <<'PY' || tail -3 gpurun_out/abp.err
import json, sys
d = json.load(open("gpurun_out/abp.json"))
p = d.get("power") or {}
pw = (p.get("power_w") or {}).get("median")
clk = (p.get("sm_mhz") or {}).get("median") or d["clocks"]["sm_mhz"]
print(*sys.argv[1:], "value", round(d["value"], 1), "MHz", clk, "per-GHz", round(d["value"] / clk * 1000, 1),
      "W", pw, "cap", (p.get("reasons_fraction") or {}).get("sw_power_cap"), "fix", d["fast_path"]["fixup_slices"])
PY
    done
  done
done
