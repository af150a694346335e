timeout 600 python tools/graph_step.py > gpurun_out/ab6_graph.jsonl 2> gpurun_out/ab6_graph.err; cat gpurun_out/ab6_graph.jsonl | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config'],d['optimizer'],d['mode'],'ms',round(d['ms'],4),'host_us',round(d['host_us_per_call'],1),'Gp/s',round(d['gparams_per_s'],1),'frac',round(d['frac_of_measured_hbm'],3))
"; tail -3 gpurun_out/ab6_graph.err
VARIANTS="base:build/base/lib.so: k0:build/k0/lib.so:" STEPS=150 REPS=3 bash tools/gpu_ab_power.sh 2>&1 | tee gpurun_out/ab6.txt
