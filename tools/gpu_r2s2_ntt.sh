mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 --e2e-reps 1 --exact-steps 0 --no-probes"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ntt_col -s 4 -c 2 -o gpurun_out/ntt_prof -f $CMD > gpurun_out/ntt_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/ntt_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ntt_src.csv 2>/dev/null
ncu -i gpurun_out/ntt_prof.ncu-rep --page raw --csv > gpurun_out/ntt_raw.csv 2>/dev/null; echo done
