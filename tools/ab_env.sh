#!/bin/bash
# A/B of an environment switch on the headline solve: alternating gap_probe runs (IPR_TIMELINE=1).
# usage: tools/ab_env.sh VAR valueA valueB [rounds]
var=$1; a=$2; b=$3; rounds=${4:-3}
for r in $(seq 1 $rounds); do
  for v in $a $b; do
    echo "== $var=$v round $r"
    env $var=$v IPR_TIMELINE=1 python tools/gap_probe.py --reps 3 2>&1 | grep -E "^ipr timeline|^rep [12]" | tail -4
  done
done
