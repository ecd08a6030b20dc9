#!/bin/bash
# one line per binary: name, occupancy, time, status
for b in tools/experiments/pipe_bin/p_*; do
  out=$(timeout 120 $b 2>&1)
  occ=$(echo "$out" | grep -o "occ=[0-9]*" | head -1)
  t=$(echo "$out" | grep "^time" | awk '{print $2}')
  ok=$(echo "$out" | tail -1 | awk '{print $NF}')
  echo "$(basename $b) $occ $t $ok"
done
