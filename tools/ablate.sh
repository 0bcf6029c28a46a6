#!/bin/bash
# Build timing-only ablation variants of libpslb200.so into build_ablate/
# (results are NOT correct; for time attribution only).
#   bash tools/ablate.sh NAME=FLAG[,FLAG] ...
cd "$(dirname "$0")/.." || exit 1
mkdir -p build_ablate
S=paper_2107_09801_b200/csrc
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  D=""; for f in ${flags//,/ }; do [ "$f" != none ] && D="$D -D$f"; done
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -shared $D \
    $S/psl_kernels.cu $S/psl_ntt.cu $S/psl_api.cu -o build_ablate/lib_$name.so &
done
wait
ls -la build_ablate
