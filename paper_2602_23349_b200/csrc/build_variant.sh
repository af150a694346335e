#!/bin/bash
# Build an experimental variant of the library: build_variant.sh <outdir> <extra nvcc flags...>
# (tile size / occupancy sweeps; the product build is the Makefile.)
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
OUT=$1; shift
mkdir -p "$OUT"
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -I$HERE/../../include -Xptxas -v"
for f in fo_step fo_step_adamw fo_step_sgd fo_step_lion fo_step_adamw_extra fo_step_sgd_extra fo_step_lion_extra fo_codec fo_host fo_api fo_selftest fo_sweep; do
  /usr/local/cuda/bin/nvcc $FLAGS "$@" -c "$HERE/$f.cu" -o "$OUT/$f.o" 2> "$OUT/$f.ptxas.log" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/lib.so" "$OUT"/fo_step.o "$OUT"/fo_step_adamw.o "$OUT"/fo_step_sgd.o "$OUT"/fo_step_lion.o "$OUT"/fo_step_adamw_extra.o "$OUT"/fo_step_sgd_extra.o "$OUT"/fo_step_lion_extra.o "$OUT"/fo_codec.o "$OUT"/fo_host.o "$OUT"/fo_api.o "$OUT"/fo_selftest.o "$OUT"/fo_sweep.o -lcudart_static -Xcompiler -fPIC
grep -A4 "Compiling entry function '_ZN2fo15step_tma_kernelILi1E13__nv_bfloat16Li384ELi0" "$OUT/fo_step_adamw.ptxas.log" | grep -E "Used|spill" | tr '\n' ' '; echo
