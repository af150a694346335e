timeout 900 python -m pytest tests/test_gpu_torch_optim.py -q -k "release" 2>&1 | tail -1
for c in 0 74 37 16; do timeout 600 python tools/bench_gpt2_train.py --modes flash_release --release-ctas $c > gpurun_out/rel_$c.jsonl 2>/dev/null; python3 -c "
import json; d=json.loads(open('gpurun_out/rel_$c.jsonl').read().strip().splitlines()[-1]); print('ctas $c', round(d['tokens_per_s']), 'opt_ms', d['optimizer_step_ms'])"; done
timeout 600 python tools/bench_gpt2_train.py --modes flash > gpurun_out/rel_deferred.jsonl 2>/dev/null; python3 -c "
import json; d=json.loads(open('gpurun_out/rel_deferred.jsonl').read().strip().splitlines()[-1]); print('deferred', round(d['tokens_per_s']), 'opt_ms', d['optimizer_step_ms'])"
