# round 2 (second session) measurements: tests, smoke, bench, reference arm, throughput, launch list, ncu
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/fin_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/fin_pytest.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/fin_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo bench=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo ref=$?
rm -f gpurun_out/fin_throughput.jsonl gpurun_out/fin_small.jsonl
for L in 16383 32767 65535 131071 262143 524287 1048575; do
  timeout 600 python tools/step_time.py --length $L --walks 444 --steps 10 --mode both >> gpurun_out/fin_throughput.jsonl 2>/dev/null
done
timeout 600 python tools/step_time.py --length 1048575 --walks 444 --steps 4 --mode auto --n-lmt 6912 >> gpurun_out/fin_throughput.jsonl 2>/dev/null
timeout 900 python tools/small_l.py --length 16383 32767 65535 131071 262143 524287 1048575 --walks 444 --steps 10 > gpurun_out/fin_small.jsonl 2>/dev/null; echo small=$?
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 --exact-steps 0"
$CMD > gpurun_out/fin_plain.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv $CMD > gpurun_out/fin_launches_run.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -s 3 -c 1 \
    -o gpurun_out/fin_prof -f $CMD > gpurun_out/fin_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/fin_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/fin_src.csv 2>/dev/null; echo src=$?
