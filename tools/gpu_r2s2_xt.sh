mkdir -p gpurun_out
timeout 600 python tools/small_l.py --length 1048575 --walks 148 444 --steps 10 > gpurun_out/x_small.jsonl 2> gpurun_out/x_small.err; echo small=$?
cat gpurun_out/x_small.jsonl
timeout 600 python -m pytest tests -q -m gpu -x -k "certcheck or phase2" 2>&1 | tail -2
