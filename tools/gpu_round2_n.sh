mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/n_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/n_pytest.log
python bench.py --no-cpu-baseline > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err; echo bench=$?
python bench.py --no-cpu-baseline > gpurun_out/n_bench2.json 2> gpurun_out/n_bench2.err; echo bench=$?
