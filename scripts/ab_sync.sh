#!/bin/bash
# host turnaround of the pipelined run loop: rounds enqueued per host check (run under gpurun)
for r in 1 2; do for c in 6 16 48; do
  echo -n "rounds/sync $c: "; GP_ROUNDS_PER_SYNC=$c timeout 300 python scripts/quick_run.py 5 | grep rep1 | sed -E 's/.*dev_ms=([0-9.]+) commit=([0-9.]+) prop=([0-9.]+) setup=([0-9.]+).*/dev \1 commit \2 prop \3 setup \4/'
done; done
