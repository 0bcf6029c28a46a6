mkdir -p gpurun_out
for L in 1048575; do
  PSLB200_LIB=build_ablate/lib_pt.so timeout 300 python tools/pt_run.py 10 $L > gpurun_out/pt2_$L.log 2>&1; echo pt$L=$?
done
