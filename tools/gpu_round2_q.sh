mkdir -p gpurun_out
timeout 700 python tools/quality.py --m 16 --seconds 120 --ablation > gpurun_out/q_m16_120s.jsonl 2> gpurun_out/q_m16.err; echo q16=$?
timeout 1200 python tools/quality.py --m 17 --seconds 300 --ablation > gpurun_out/q_m17_300s.jsonl 2> gpurun_out/q_m17.err; echo q17=$?
timeout 2100 python tools/quality.py --m 18 --seconds 600 --ablation > gpurun_out/q_m18_600s.jsonl 2> gpurun_out/q_m18.err; echo q18=$?
