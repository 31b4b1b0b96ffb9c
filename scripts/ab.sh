#!/bin/bash
# A/B two prebuilt libraries on config $1, $2 reps each (dev helper)
for r in $(seq 1 $2); do
  for v in old new; do
    cp abso/$v.so paper_2007_16076_b200/libgeopairs_b200.so
    echo -n "$v "; timeout 300 python scripts/quick_run.py $1 | grep rep1 | sed -E 's/.*dev_ms=([0-9.]+) commit=([0-9.]+) prop=([0-9.]+).*/dev \1 commit \2 prop \3/'
  done
done
