#!/bin/bash
# Full ncu capture (one per gpurun call) of the dominant kernel of a bench configuration.
# Usage (repo root, under gpurun): bash tools/ncu_full.sh <tag> <kernel-regex> [bench args...]
set -u
tag=$1; kre=$2; shift 2
out=gpurun_out/$tag
mkdir -p $out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o $out/prof \
  python bench.py --no-cpu-baseline --no-e2e --min-seconds 0 "$@" > $out/ncu_full.log 2>&1; echo "ncu full rc=$?"
