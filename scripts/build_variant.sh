#!/bin/bash
# build_variant.sh NAME "-DFOO=1 ..." [sources...]: the library with extra
# defines on the given csrc sources (default: all .cu) into _variants/NAME/
# for scripts/gpu_variants.sh A/B runs (development aid).
set -e
name=$1; defs=$2; shift 2
here=$(cd "$(dirname "$0")/.." && pwd)
pkg=$here/paper_2405_00698_b200
make -C "$pkg" -j8 > /dev/null
out=$here/_variants/$name
rm -rf "$out"; mkdir -p "$out/obj"
cp "$pkg"/build/*.o "$out/obj/"
srcs=${@:-$(cd "$pkg/csrc" && ls *.cu)}
for s in $srcs; do
  rdc=""; [ "$s" = integrator_cluster.cu ] && rdc="-rdc=true"  # device-launched filler (Makefile)
  /usr/local/cuda/bin/nvcc $rdc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC -ccbin /usr/bin/g++ -Xptxas -v --expt-relaxed-constexpr -I"$here/include" -DVX_BUILDING $defs \
    -c "$pkg/csrc/$s" -o "$out/obj/${s%.cu}.o" > "$out/${s%.cu}.ptxas.log" 2>&1 || { cat "$out/${s%.cu}.ptxas.log"; exit 1; }
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -rdc=true -shared -ccbin /usr/bin/g++ -o "$out/libvoxevo_b200.so" "$out"/obj/*.o -lcudadevrt -lpthread
rm -rf "$out/obj"
echo "built $out"
