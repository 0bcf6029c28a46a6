mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo smoke=$?
timeout 600 python tools/deep_starts.py > gpurun_out/c_deep.log 2>&1; echo deep=$?
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/c_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/c_bench.log 2>&1; echo bench=$?
