#!/bin/bash
# Convert ncu reports under gpurun_out/ to text summaries (details page, raw CSV)
# and drop the binary reports (gpurun copies back <= 64 MiB).
for r in gpurun_out/*.ncu-rep; do
  [ -e "$r" ] || continue
  b="${r%.ncu-rep}"
  ncu -i "$r" --page details > "$b.details.txt" 2>&1
  ncu -i "$r" --page raw --csv > "$b.raw.csv" 2>&1
  gzip -f "$b.raw.csv"
  rm -f "$r"
done
