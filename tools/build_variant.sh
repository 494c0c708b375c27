#!/bin/bash
# Build the library with extra compile flags into tools/ab/lib_NAME.so (timing
# A/B of build-time variants, tools/sym_ab.py), then rebuild the default.
# usage: tools/build_variant.sh NAME "-DNCGP_X=1 ..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2310_20285_b200/csrc
mkdir -p $ROOT/tools/ab
rm -f $C/build/kop_tc.o
make -C $C -j8 EXTRA="$2" >/dev/null
cp $ROOT/paper_2310_20285_b200/libncgp_b200.so $ROOT/tools/ab/lib_$1.so
rm -f $C/build/kop_tc.o
make -C $C -j8 >/dev/null
