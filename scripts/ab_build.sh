#!/bin/bash
# Cross-compiles compile-time variants of libsfcnl_b200.so into abv/<name>/ (git- and
# not gpurun-ignored): ab_build.sh name1 "EXTRA flags" name2 "EXTRA flags" ...
# then on the box: for v in abv/*; do SFCNL_LIB=$v/libsfcnl_b200.so python scripts/stage_times.py; done
set -e
cd "$(dirname "$0")/../paper_2602_19873_b200"
while [ $# -ge 2 ]; do
  name=$1; extra=$2; shift 2
  make -s OBJ=build_$name EXTRA="$extra" -j16 libsfcnl_b200.so 2>&1 | grep -E "error" || true
  mkdir -p ../abv/$name && mv libsfcnl_b200.so ../abv/$name/
  rm -rf "build_$name"  # variant objects (would bloat the gpurun snapshot)
done
make -s -j16 libsfcnl_b200.so
