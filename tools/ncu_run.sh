# one full ncu capture of the dominant kernel (run_kernel) from the bench command
ARGS="--steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 $*"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:run_kernel -s 1 -c 1 -o gpurun_out/prof_run -f python bench.py $ARGS > gpurun_out/ncu.log 2>&1
