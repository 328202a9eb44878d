# round 2, run 97: rebuilt library (source as validated in run 92) -- smoke + GPU suite
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_97_smoke.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_97_pytest.txt 2>&1
