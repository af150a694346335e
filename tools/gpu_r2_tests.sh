# round 2: full GPU test suite, smoke, headline bench
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2_pytest.txt 2>&1; tail -5 gpurun_out/r2_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -2 gpurun_out/r2_smoke.txt
