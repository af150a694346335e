# parity stress on the final build (both launches programmatic)
python tools/parity_stress.py --seconds 480 --seed 21 > gpurun_out/stress_f2.json 2> gpurun_out/stress_f2.err; tail -1 gpurun_out/stress_f2.json
python tools/parity_stress.py --seconds 240 --seed 22 --layouts > gpurun_out/stress_f2_layouts.json 2> gpurun_out/stress_f2_layouts.err; tail -1 gpurun_out/stress_f2_layouts.json
