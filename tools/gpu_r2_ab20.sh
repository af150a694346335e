# persistent grid on fewer SMs under the 1000 W limit (FO_GRID_SMS), Llama-8B AdamW
for rep in 1 2; do for k in 148 140 132 120; do
  FO_GRID_SMS=$k timeout 300 python bench.py --steps 150 --warmup 5 --no-e2e --no-cpu --no-parity > gpurun_out/ab20.json 2> gpurun_out/ab20.err
  python3 - "$k" <<'PY' || tail -3 gpurun_out/ab20.err
import json, sys
d = json.load(open("gpurun_out/ab20.json"))
p = d.get("power") or {}
clk = (p.get("sm_mhz") or {}).get("median") or d["clocks"]["sm_mhz"]
print("sms", sys.argv[1], "capped", round(d["value"], 1), "MHz", clk, "W", (p.get("power_w") or {}).get("median"),
      "single", round(d["single_launch_after_idle"]["gparams_s"], 1))
PY
done; done
