#!/bin/bash
# Builds an experimental variant of the product library with extra -D flags into
# diag/_variants/<name>/libgsmap_b200.so (selected at run time by GSMAP_B200_VARIANT=<name>).
#   diag/build_variant.sh fwd9 -DGSB_FWD_MIN_BLOCKS=9
set -e
name=$1; shift
here=$(cd "$(dirname "$0")" && pwd)
src=$here/../paper_2411_02703_b200/csrc
out=$here/_variants/$name
mkdir -p "$out/obj"
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Wno-deprecated-declarations -Xptxas -v $*"
pids=()
for f in comm sort raster blend_fwd blend_bwd loss adam host host_mapping host_io microbench; do
  nvcc $FLAGS -c "$src/$f.cu" -o "$out/obj/$f.o" 2> "$out/obj/$f.ptxas.log" & pids+=($!)
done
nvcc $FLAGS --fmad=false -c "$src/geometry.cu" -o "$out/obj/geometry.o" 2> "$out/obj/geometry.ptxas.log" & pids+=($!)
for p in "${pids[@]}"; do wait $p; done
nvcc $ARCH -shared -o "$out/libgsmap_b200.so" "$out"/obj/*.o -Xcompiler -fPIC -ldl
echo "built $out/libgsmap_b200.so"
