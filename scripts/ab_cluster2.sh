#!/bin/bash
set -u
timeout 300 python -m pytest tests/test_gpu_edge.py -q -x -k cluster 2>&1 | tail -1
for env in "GP_PROP_CLUSTER=1" "GP_PROP_CLUSTER=1 GP_DELTA_FACTOR=48" "GP_PROP_CLUSTER=1 GP_DELTA_FACTOR=inf" "GP_PROP_CLUSTER=0 GP_DELTA_FACTOR=48"; do
  echo "== $env"
  env GP_CL_DEBUG=1 $env timeout 300 python scripts/quick_run.py 5 2>&1 | tail -2
done
