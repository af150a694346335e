timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab7_tests.txt 2>&1; tail -2 gpurun_out/ab7_tests.txt
for v in base new; do lib=build/base/lib.so; [ $v = new ] && lib=paper_2602_23349_b200/libflashoptim_b200.so
for rep in 1 2; do FO_LIB_PATH=$PWD/$lib timeout 600 python tools/graph_step.py > gpurun_out/ab7_graph_$v.jsonl 2>/dev/null; python3 -c "
import sys,json
for l in open('gpurun_out/ab7_graph_$v.jsonl'):
    d=json.loads(l); print('$v', d['config'],d['optimizer'],d['mode'],'ms',round(d['ms'],4),'Gp/s',round(d['gparams_per_s'],1),'frac',round(d['frac_of_measured_hbm'],3))
"; done; done
