#!/bin/bash
# Throughput at m14..m20 (bench.py per length) and best PSL at fixed wall time
# (tools/quality.py, two-phase + single-exponent ablations), one B200.
mkdir -p gpurun_out
for L in 16383 65535 262143 1048575; do
  timeout 600 python bench.py --length $L --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/sweep.jsonl
done
timeout 600 python bench.py --n-lmt 6912 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/sweep.jsonl
timeout 1500 python tools/quality.py --m 14 15 16 17 18 19 20 --seconds 30 --ablation > gpurun_out/quality.jsonl 2> gpurun_out/quality.err
echo sweep done
