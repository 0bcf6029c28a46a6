set -x
mkdir -p gpurun_out
nvidia-smi -L; nproc; lscpu | head -20 > gpurun_out/lscpu.txt
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
for t in memcheck racecheck synccheck; do
  for cfg in "2048 auto" "5000 auto" "2048 exact"; do
    timeout 600 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py $cfg > "gpurun_out/san_${t}_${cfg// /_}.log" 2>&1; echo "$t $cfg = $?"
  done
done
