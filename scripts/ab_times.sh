#!/bin/bash
# Same-box A/B of decode-kernel variants: for each build/ab/<name>.so, the
# config-4 step's kernel times and the per-chain decode times of the chains named
# in $CHAINS (default: the slowest config-4 chains).  usage: scripts/ab_times.sh name...
CHAINS=${CHAINS:-33,51,63,46,26,41,57,36}
CFG=${CFG:-4}
for n in "$@"; do
  echo "== $n"
  GL_LIB_PATH=build/ab/$n.so python scripts/quick_times.py $CHAINS $CFG
done
