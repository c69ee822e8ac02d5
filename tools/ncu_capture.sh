#!/bin/bash
# ncu --set full of ONE launch of each kernel regex given, on a bench command.
# Writes text only (raw metrics CSV + source-line CSV) to $OUT (default
# gpurun_out/ncu); the .ncu-rep files stay in /tmp (they exceed gpurun's
# 64 MiB copy-back limit).
#   tools/ncu_capture.sh <tag> "<bench args>" kregex1 [kregex2 ...]
set -u
TAG=$1; shift
ARGS=$1; shift
OUT=${OUT:-gpurun_out/ncu}
mkdir -p "$OUT" /tmp/ncu
for K in "$@"; do
  R=/tmp/ncu/${TAG}_${K}
  ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 -f -o "$R" \
      python bench.py $ARGS > /dev/null 2>&1
  ncu -i "$R.ncu-rep" --page raw --csv > "$OUT/${TAG}_${K}_raw.csv" 2>/dev/null
  ncu -i "$R.ncu-rep" --page source --csv --print-source sass > "$OUT/${TAG}_${K}_sass.csv" 2>/dev/null
  ncu -i "$R.ncu-rep" --page details --csv > "$OUT/${TAG}_${K}_details.csv" 2>/dev/null
done
