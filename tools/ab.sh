#!/bin/bash
# A/B timing of in-tree library variants: tools/ab.sh tagA tagB ... (libfks_<tag>.so), 3 rounds
for r in 1 2 3; do
  for v in "$@"; do
    echo -n "$v: "; FKS_LIB_VARIANT=$v python tools/quick_time.py 2>&1 | grep -E "C1|C2"
  done
done
