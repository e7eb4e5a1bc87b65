#!/bin/bash
# Build a library variant with extra nvcc defines, for A/B timing (tools/ab_lib.sh).
# usage: tools/build_variant.sh NAME "-DVG_FOO=1 -DVG_BAR=2"  -> paper_2202_00242_b200/lib/NAME.so
set -e
cd "$(dirname "$0")/.."
make -j8 LIB=paper_2202_00242_b200/lib/$1.so OBJDIR=build/var_$1 EXTRA_NVFLAGS="$2" >/dev/null
echo "built paper_2202_00242_b200/lib/$1.so ($2)"
