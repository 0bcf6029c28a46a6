N=paper_2107_09801_b200/libpslb200.so
python tools/ab_time.py $N build_ablate/lib_xev.so 3 2>&1 | tail -2
python tools/ab_time.py $N build_ablate/lib_aeo.so 3 2>&1 | tail -2
