#!/bin/bash
# build a tuning variant of the library: tools/build_variant.sh <name> "<-D flags>"
# -> paper_1201_2936_b200/variants/<name>.so (select with SH_LIB=...)
set -e
cd "$(dirname "$0")/../paper_1201_2936_b200/csrc"
mkdir -p ../variants
make -s OUT=../variants/$1.so EXTRA="$2" ../variants/$1.so
grep -A2 "k_stream" build.log | grep -E "registers|spill" | head -8
