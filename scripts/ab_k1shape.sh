#!/bin/bash
# K1 CTA shapes at 256^2 (run under gpurun)
for env in "GP_PROP_THREADS=512 GP_PROP_MINB=3" "GP_PROP_THREADS=768 GP_PROP_MINB=2" "GP_PROP_THREADS=384 GP_PROP_MINB=4"; do
  echo "== $env"; env $env timeout 300 python scripts/quick_run.py 5 2>&1 | tail -1
done
