#!/bin/bash
# Developer A/B builds: tools/variant.sh NAME "-DFOO=1 ..." file.cu [file.cu ...]
# recompiles the named sources with the extra defines and links them with the
# product objects (lib/obj) into lib/NAME/libfsvd_b200.so (select it with
# FSVD_LIB=paper_2508_01506_b200/lib/NAME/libfsvd_b200.so).
set -e
cd "$(dirname "$0")/../paper_2508_01506_b200/csrc"
make -s -j16 >/dev/null
name=$1; defs=$2; shift 2
out=../lib/$name; mkdir -p $out/obj
objs=""
for f in common planes gemm_tc gemm_ln_tc gemm_ln2_tc attn_tc decode ffn_tc ffn2_tc ffn_wide_tc simt runtime model_file factorize capi; do
  if printf '%s\n' "$@" | grep -qx "$f.cu"; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I../../include $defs -c -o $out/obj/$f.o $f.cu &
    objs="$objs $out/obj/$f.o"
  else
    objs="$objs ../lib/obj/$f.o"
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libfsvd_b200.so $objs -Xcompiler -fvisibility=hidden
echo "built $out/libfsvd_b200.so ($defs)"
