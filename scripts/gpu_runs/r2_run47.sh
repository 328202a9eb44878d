# round 2, run 47: compute-sanitizer memcheck over small GPU tests (kernels of
# every family), racecheck / synccheck on the shared-memory-staged pass and pair paths
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_io.py tests/test_collapse_cas.py tests/test_ppr.py -q -m gpu -x -k "not big and not c4 and not aucroc" > gpurun_out/r2_47_memcheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_47_racecheck.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_47_synccheck.txt 2>&1
