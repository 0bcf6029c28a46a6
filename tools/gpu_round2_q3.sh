mkdir -p gpurun_out
timeout 3300 python tools/quality.py --m 20 --seconds 2400 --modes two-phase > gpurun_out/q3_m20_2400s.jsonl 2> gpurun_out/q3.err; echo q20=$?
