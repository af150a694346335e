# final check on the PDL build + same-box A/B of GPT-2-medium training with gradient release (pdlA = in-tree vs pdl0)
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_pdl.py -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for rep in 1 2 3; do for v in pdlA pdl0; do FO_LIB_PATH=$PWD/build/$v/lib.so timeout 600 python tools/bench_gpt2_train.py --modes flash,flash_release --steps 20 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$v', d['mode'], round(d['tokens_per_s']), round(d['ms_per_step'],2), round(d['optimizer_step_ms'],3))
"; done; done
