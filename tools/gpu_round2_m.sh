mkdir -p gpurun_out
timeout 1200 python tools/chain.py --m 16 --rounds 4 --seconds 120 > gpurun_out/m_chain_m16.jsonl 2> gpurun_out/m_chain.err; echo chain=$?
