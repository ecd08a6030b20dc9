#!/bin/bash
for b in tools/experiments/rows_bin/c_*; do
  echo "== $b"
  timeout 120 $b "$@" 2>&1 | tail -3
done
