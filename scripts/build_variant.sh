#!/bin/bash
# Build an A/B variant of libotprg.so: scripts/build_variant.sh NAME "EXTRA_NVFLAGS" [file=replacement ...]
# -> paper_2203_03732_b200/lib/libotprg_NAME.so (sources copied to /tmp, the tree is untouched)
set -e
NAME=$1; EXTRA=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d /tmp/otprg_var_XXXX)
mkdir -p $T/pkg $T/include
cp -r $ROOT/paper_2203_03732_b200/csrc $T/pkg/
cp $ROOT/include/* $T/include/
for kv in "$@"; do f=${kv%%=*}; r=${kv#*=}; cp "$r" $T/pkg/csrc/$f; done
make -s -C $T/pkg/csrc NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xptxas -v -Xcompiler -fPIC,-ffp-contract=off,-O2 -I$T/include $EXTRA" >/dev/null 2>&1 || { echo "build failed"; exit 1; }
mkdir -p $ROOT/paper_2203_03732_b200/lib
cp $T/pkg/lib/libotprg.so $ROOT/paper_2203_03732_b200/lib/libotprg_$NAME.so
rm -rf $T
echo built libotprg_$NAME.so
