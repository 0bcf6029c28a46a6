mkdir -p gpurun_out
export PSLB200_LIB=build_ablate/lib_bounds.so
timeout 2400 python -m pytest tests -q -m gpu --deselect tests/test_dropin.py -p no:cacheprovider > gpurun_out/f_bounds_pytest.log 2>&1; echo bounds_pytest=$?
for cfg in "2048 auto" "5000 auto" "2048 exact" "70000 auto" "300000 auto"; do
  timeout 600 python tools/sanitize_run.py $cfg 12 >> gpurun_out/f_bounds_runs.log 2>&1; echo "run $cfg = $?"
done
unset PSLB200_LIB
for L in 16383 65535; do timeout 300 python tools/step_time.py --length $L --walks 444 --steps 20 --mode both >> gpurun_out/f_smallL.log 2>&1; done
timeout 900 python tools/deep_starts.py 60000 0 25000 > gpurun_out/f_deep.log 2>&1; echo deep=$?
