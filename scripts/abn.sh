#!/bin/bash
# run config $1 with each prebuilt library abso/<name>.so given as further args (dev helper)
c=$1; shift
for v in "$@"; do
  cp abso/$v.so paper_2007_16076_b200/libgeopairs_b200.so
  echo -n "$v "; timeout 300 python scripts/quick_run.py $c | grep rep1 | sed -E 's/.*dev_ms=([0-9.]+) commit=([0-9.]+) prop=([0-9.]+).*/dev \1 commit \2 prop \3/'
done
