# bounds-check build (PSL_DEBUG_BOUNDS) through the GPU suite and small sanitizer-style runs
mkdir -p gpurun_out
export PSLB200_LIB=build_ablate/lib_bounds.so
timeout 2400 python -m pytest tests -q -m gpu --deselect tests/test_dropin.py -p no:cacheprovider > gpurun_out/s2_bounds_pytest.log 2>&1; echo bounds_pytest=$?
tail -2 gpurun_out/s2_bounds_pytest.log
rm -f gpurun_out/s2_bounds_runs.log
for cfg in "2048 auto" "5000 auto" "2048 exact" "70000 auto" "300000 auto"; do
  timeout 600 python tools/sanitize_run.py $cfg 12 >> gpurun_out/s2_bounds_runs.log 2>&1; echo "run $cfg = $?"
done
unset PSLB200_LIB

