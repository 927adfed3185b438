#!/bin/bash
# A/B builds of libmargingate with extra -D flags (diagnostic only):
#   scripts/build_variant.sh NAME [-DFLAG=V ...]  ->  scripts/ab/libNAME.so
# Used with MG_LIB_PATH=scripts/ab/libNAME.so python scripts/ab_step.py ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/scripts/ab/$name
mkdir -p "$out"
objs=()
for f in gemm elementwise attention control engine capi_debug; do
  [ -f "$root/paper_2605_30218_b200/csrc/$f.cu" ] || continue
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I"$root/include" "$@" -c "$root/paper_2605_30218_b200/csrc/$f.cu" -o "$out/$f.o" &
  objs+=("$out/$f.o")
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/scripts/ab/lib$name.so" "${objs[@]}" \
  -lcudart_static -ldl -lrt -lpthread
echo "built scripts/ab/lib$name.so"
