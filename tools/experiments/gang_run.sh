#!/bin/bash
# run every built gang bench instance (timeout per run)
mkdir -p gpurun_out
for b in tools/experiments/gang_bin/g_*; do
  echo "== $b"
  timeout 60 $b "$@" 2>&1 | tail -6
done
