#!/bin/bash
# Builds ab/libdynmo_stamps.so: the library with -DDYNMO_STEP_STAMPS (per
# kernel first-warp start / last-warp end, read by tools/step_stamps.py).
set -e
cd "$(dirname "$0")/../paper_2505_14864_b200/csrc"
make -s
ARCH="-gencode arch=compute_100a,code=sm_100a"
NCCL=$(python -c "import nvidia.nccl, os; print(os.path.dirname(nvidia.nccl.__file__))" 2>/dev/null || echo /opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl)
T=$(mktemp -d)
for f in k_profile k_solve; do
  nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -I../../include -I. -I$NCCL/include -DDYNMO_STEP_STAMPS \
    $( [ $f = k_solve ] && echo -fmad=false ) -c $f.cu -o $T/$f.o 2>/dev/null
done
nvcc $ARCH -O3 -std=c++17 -Xcompiler -fPIC -I../../include -I. -I$NCCL/include -DDYNMO_STEP_STAMPS -x cu -c dynmo_host.cpp -o $T/dynmo_host.o
mkdir -p ../../ab
nvcc $ARCH -shared -o ../../ab/libdynmo_stamps.so $(ls build/*.o | grep -v "k_solve.o\|k_profile.o\|dynmo_host.o") $T/*.o \
  -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
echo built ab/libdynmo_stamps.so
