# round 2 session 2: source-level ncu capture of the certified kernel + small-L launch shapes
mkdir -p gpurun_out
timeout 600 python tools/small_l.py --length 16383 65535 --walks 148 444 888 --steps 20 > gpurun_out/p_small.jsonl 2> gpurun_out/p_small.err; echo small=$?
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --exact-steps 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -s 3 -c 1 \
    -o gpurun_out/p_prof -f python bench.py $ARGS > gpurun_out/p_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/p_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/p_src.csv 2>/dev/null; echo src=$?
ncu -i gpurun_out/p_prof.ncu-rep --page raw --csv > gpurun_out/p_raw.csv 2>/dev/null; echo raw=$?
