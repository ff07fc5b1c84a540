#!/bin/bash
# Build libmppi_b200 from git revision $1 into $2 (A/B perf comparisons; not part of the library).
set -e
REV=$1; OUT=$2; shift 2
D=$(mktemp -d)
git -C /root/repo archive $REV paper_2603_07199_b200/csrc include | tar -x -C $D
NCCL=$(python -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])")
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared "$@" \
  -I $NCCL/include -I $D/include $D/paper_2603_07199_b200/csrc/*.cu -L $NCCL/lib -l:libnccl.so.2 \
  -Xlinker=-rpath=$NCCL/lib -o $OUT
rm -rf $D
