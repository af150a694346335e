#!/bin/bash
# guard-mode A/B: build/a (FO_VG=0, gradient guard) vs build/b (FO_VG=1,
# operand guards): parity tests through each, headline per GHz for all three
# optimizers, planted tiny gradients and the GPT-2 training step.
for lib in build/a/lib.so build/b/lib.so; do
  echo "== tests $lib"
  FO_LIB_PATH=$PWD/$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_g32.py -x -q 2>&1 | tail -3
done
for o in adamw sgd lion; do OPT=$o timeout 900 ./tools/gpu_ab_alt.sh; done
for lib in build/a/lib.so build/b/lib.so; do
  echo "== $lib"
  FO_LIB_PATH=$PWD/$lib timeout 600 python tools/fallback_cost.py 2>&1 | grep -v Warn | tail -7
  FO_LIB_PATH=$PWD/$lib timeout 600 python tools/bench_gpt2_train.py --modes flash --steps 10 --warmup 5 2>&1 | python -c "import sys,json; [print((d:=json.loads(l))['mode'], round(d['tokens_per_s']), round(d['optimizer_step_ms'],3)) for l in sys.stdin if l.startswith('{')]"
done
