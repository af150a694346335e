# L2 cache-policy hints on the ring's bulk reads (h1: evict_first) and the prefetch (h2: + evict_last) vs none (base = in-tree)
mkdir -p build/base && cp paper_2602_23349_b200/libflashoptim_b200.so build/base/lib.so
for rep in 1 2; do for v in base h1 h2; do
  FO_LIB_PATH=$PWD/build/$v/lib.so timeout 300 python bench.py --steps 150 --warmup 5 --no-e2e --no-cpu --no-parity > gpurun_out/ab19.json 2> gpurun_out/ab19.err
  python3 - "$v" <<'PY' || tail -3 gpurun_out/ab19.err
import json, sys
d = json.load(open("gpurun_out/ab19.json"))
p = d.get("power") or {}
clk = (p.get("sm_mhz") or {}).get("median") or d["clocks"]["sm_mhz"]
print(sys.argv[1], "capped", round(d["value"], 1), "MHz", clk, "per-GHz", round(d["value"] / clk * 1000, 1),
      "single", round(d["single_launch_after_idle"]["gparams_s"], 1))
PY
done; done
for v in base h1 h2; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 300 python tools/graph_step.py --steps 300 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if d['mode']=='launch': print('$v', d['config'], d['optimizer'], 'ms', round(d['ms'],4))
"; done
