mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests/test_gpu_certcheck.py tests/test_gpu_multi.py tests/test_dropin.py -q -m gpu > gpurun_out/b_new.log 2>&1; echo new=$?
timeout 900 python bench.py > gpurun_out/b_bench.log 2>&1; echo bench=$?
timeout 1500 python -m pytest tests -q -m gpu --deselect tests/test_gpu_certcheck.py --deselect tests/test_gpu_multi.py --deselect tests/test_dropin.py > gpurun_out/b_pytest.log 2>&1; echo pytest=$?
