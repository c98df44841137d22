#!/bin/bash
# Build an experiment variant of libemie_cu.so: tools/build_variant.sh OUTDIR -DFLAG=...
set -e
out=$1; shift
cd "$(dirname "$0")/../paper_1512_06126_b200/csrc"
mkdir -p "$out"
objs=()
for s in capi.cu operator.cu lateral.cu solver.cu greens.cu shard.cu peer.cu dense.cu layered.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
    -I ../../include --expt-relaxed-constexpr "$@" -c $s -o "$out/$s.o" &
  objs+=("$out/$s.o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libemie_cu.so" "${objs[@]}" -cudart static
rm -f "$out"/*.o
