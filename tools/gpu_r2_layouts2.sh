timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/lay2_tests.txt 2>&1; tail -3 gpurun_out/lay2_tests.txt
timeout 400 python tools/parity_stress.py --seconds 300 --seed 11 --layouts > gpurun_out/lay2_stress.json 2>&1; tail -1 gpurun_out/lay2_stress.json
timeout 600 python tools/bench_variants.py --config gpt2_medium > gpurun_out/lay2_var_gpt2.jsonl 2>&1
timeout 900 python tools/bench_variants.py --config llama31_8b --steps 5 > gpurun_out/lay2_var_llama.jsonl 2>&1
for o in sgd lion; do timeout 600 python tools/bench_variants.py --config gpt2_medium --optimizer $o >> gpurun_out/lay2_var_gpt2.jsonl 2>&1; done
python3 -c "
import json
for f in ['gpurun_out/lay2_var_gpt2.jsonl','gpurun_out/lay2_var_llama.jsonl']:
    for l in open(f):
        try: d=json.loads(l)
        except Exception: continue
        print(d['config'], d['optimizer'], d['variant'], d['kernel'], round(d['gparams_per_s'],1), round(d['frac_of_measured_hbm'],3))
"
