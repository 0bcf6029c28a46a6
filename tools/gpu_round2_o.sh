mkdir -p gpurun_out
nproc; python -c "
import numpy as np, time
a=np.ones(444*1048575, np.int8); b=np.empty_like(a)
for i in range(3):
    t=time.time(); np.copyto(b,a); print('memcpy 444MB %.1f ms'%(1e3*(time.time()-t)))
"
echo old; NW=444 PSLB200_LIB=build_ablate/lib_nostag2.so python tools/e2e_breakdown.py 10
echo new; NW=444 python tools/e2e_breakdown.py 10
