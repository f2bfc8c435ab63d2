#!/bin/bash
# A/B of an engine env switch on device time: tools/ab_env.sh "ITERCUR_PDL=1" 4 3 5
sw="$1"; shift
for c in "$@"; do
  echo "== config $c default"; timeout 600 python tools/time_runs.py --config $c --runs 8 | awk '{printf "%s ", $4} END {print ""}'
  echo "== config $c $sw"; env $sw timeout 600 python tools/time_runs.py --config $c --runs 8 | awk '{printf "%s ", $4} END {print ""}'
done
