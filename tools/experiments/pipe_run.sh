#!/bin/bash
for b in tools/experiments/pipe_bin/p_*; do
  echo "== $b"
  timeout 120 $b "$@" 2>&1 | tail -4
done
