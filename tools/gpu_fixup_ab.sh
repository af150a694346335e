#!/bin/bash
# A/B of build/a vs build/b: headline (alternating twice), planted tiny
# gradients (tools/fallback_cost.py) and the GPT-2 training step.
OPT=adamw timeout 900 ./tools/gpu_ab_alt.sh
for lib in build/a/lib.so build/b/lib.so; do
  echo "== $lib"
  FO_LIB_PATH=$PWD/$lib timeout 600 python tools/fallback_cost.py 2>&1 | grep -v Warn | tail -8
  FO_LIB_PATH=$PWD/$lib timeout 600 python tools/bench_gpt2_train.py --modes flash --steps 10 --warmup 5 2>&1 | python -c "import sys,json; [print((d:=json.loads(l))['mode'], round(d['tokens_per_s']), round(d['optimizer_step_ms'],3), d['optimizer_step_back_to_back']) for l in sys.stdin if l.startswith('{')]"
done
