mkdir -p gpurun_out
timeout 2100 python tools/quality.py --m 19 --seconds 1800 --modes ${MODE} > gpurun_out/q4_m19_${MODE}_1800s.jsonl 2> gpurun_out/q4_${MODE}.err; echo q19=$?
