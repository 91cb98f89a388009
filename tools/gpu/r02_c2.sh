OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/c2_smoke.log 2>&1; echo smoke_rc=$?; tail -5 $OUT/c2_smoke.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q > $OUT/c2_pytest.log 2>&1; echo pytest_rc=$?
tail -30 $OUT/c2_pytest.log
