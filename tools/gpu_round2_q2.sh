mkdir -p gpurun_out
timeout 400 python tools/quality.py --m 14 --seconds 60 --modes two-phase > gpurun_out/q2_m14_60s.jsonl 2> gpurun_out/q2.err; echo q14=$?
timeout 400 python tools/quality.py --m 15 --seconds 120 --modes two-phase > gpurun_out/q2_m15_120s.jsonl 2>> gpurun_out/q2.err; echo q15=$?
timeout 2200 python tools/quality.py --m 19 --seconds 1800 --modes two-phase > gpurun_out/q2_m19_1800s.jsonl 2>> gpurun_out/q2.err; echo q19=$?
timeout 3000 python tools/quality.py --m 20 --seconds 2700 --modes two-phase > gpurun_out/q2_m20_2700s.jsonl 2>> gpurun_out/q2.err; echo q20=$?
