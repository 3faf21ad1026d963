#!/bin/bash
# A/B of library variants on the C2 step (development aid): tools/ab_bench.sh <out> <variant>... ("base" = libfks.so)
cd "$(dirname "$0")/.."
out=$1; shift
for round in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then unset FKS_LIB_VARIANT; else export FKS_LIB_VARIANT=$v; fi
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-spatial-secondary > /tmp/ab_$v.json 2>/dev/null
    python -c "import json; d=json.load(open('/tmp/ab_$v.json')); print('$round $v', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])" >> $out
  done
done
unset FKS_LIB_VARIANT
