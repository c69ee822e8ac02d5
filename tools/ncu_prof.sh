#!/bin/bash
# ncu --set full of ONE launch of each kernel regex on tools/prof_run.py
# (text exports only; the .ncu-rep stays in /tmp):
#   tools/ncu_prof.sh <tag> "<prof_run args>" kregex1 [kregex2 ...]
set -u
TAG=$1; shift
ARGS=$1; shift
OUT=${OUT:-gpurun_out/ncu}
mkdir -p "$OUT" /tmp/ncu
for K in "$@"; do
  R=/tmp/ncu/${TAG}_${K}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$K" -s 2 -c 1 -f -o "$R" \
      python tools/prof_run.py $ARGS > /dev/null 2>&1
  ncu -i "$R.ncu-rep" --page raw --csv > "$OUT/${TAG}_${K}_raw.csv" 2>/dev/null
  ncu -i "$R.ncu-rep" --page source --csv --print-source sass > "$OUT/${TAG}_${K}_sass.csv" 2>/dev/null
  ncu -i "$R.ncu-rep" --page details --csv > "$OUT/${TAG}_${K}_details.csv" 2>/dev/null
done
