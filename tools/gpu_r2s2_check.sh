# round 2 session 2: re-verify the restored HEAD on a B200 (tests, smoke, bench)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s2_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo bench=$?
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/s2_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/s2_pytest.log
