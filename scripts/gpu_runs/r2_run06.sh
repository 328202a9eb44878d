# round 2, run 6: new tests (device edge-list parser, GSHG/GSHE staging,
# run-dependent CAS collapse, INTEGRATION stub, reference negatives), full GPU suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_io.py tests/test_collapse_cas.py tests/test_integration.py tests/test_eval.py -q -m gpu -x > gpurun_out/r2_06_new.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2_06_pytest.txt 2>&1
