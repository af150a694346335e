# long parity stress on the final build: default layout, then the optional layouts
python tools/parity_stress.py --seconds 1500 --seed 11 > gpurun_out/stress_long.json 2> gpurun_out/stress_long.err; tail -1 gpurun_out/stress_long.json
python tools/parity_stress.py --seconds 600 --seed 12 --layouts > gpurun_out/stress_long_layouts.json 2> gpurun_out/stress_long_layouts.err; tail -1 gpurun_out/stress_long_layouts.json
