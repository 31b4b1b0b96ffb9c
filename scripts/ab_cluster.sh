#!/bin/bash
# A/B of the cluster K1 against the single-CTA K1 (run under gpurun).
set -u
for env in "GP_PROP_CLUSTER=1" "GP_PROP_CLUSTER=0" "GP_PROP_CLUSTER=1 GP_SPEC_K=296" "GP_PROP_CLUSTER=1 GP_SPEC_K=222" "GP_PROP_CLUSTER=1 GP_SPEC_K=592"; do
  echo "== $env"
  env $env timeout 300 python scripts/quick_run.py 5 2>&1 | tail -1
done
for c in 3 4; do
  for env in "GP_PROP_CLUSTER=2" "GP_PROP_CLUSTER=1"; do
    echo "== cfg$c $env"; env $env timeout 300 python scripts/quick_run.py $c 2>&1 | tail -1
  done
done
