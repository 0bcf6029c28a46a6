mkdir -p gpurun_out
A=build_ablate/lib_bandovf.so; B=build_ablate/lib_nostag2.so; N=paper_2107_09801_b200/libpslb200.so
python tools/ab_time.py $B $N 3 > gpurun_out/j_ab20.log 2>&1
python tools/ab_time.py $B $N 3 -- --length 262143 --walks 444 --steps 10 --mode auto > gpurun_out/j_ab18.log 2>&1
python tools/ab_time.py $B $N 3 -- --length 65535 --walks 444 --steps 20 --mode auto > gpurun_out/j_ab16.log 2>&1
python tools/ab_time.py $A $B 3 > gpurun_out/j_ab20b.log 2>&1
cat gpurun_out/j_ab*.log
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/j_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/j_pytest.log
