#!/bin/bash
# A/B of config-4 knobs on one B200: each variant is one process (knobs are
# read once per process); prints one JSON line per variant.
# usage: tools/ab_config4.sh OUT "ENV1" "ENV2" ...
out=$1; shift
for v in "$@"; do
  echo "== $v" >> "$out"
  env $v timeout 900 python bench.py --config ${AB_CONFIG:-4} --iters ${AB_ITERS:-4} 2>&1 | grep '^{' | sed "s/^{/{\"env\": \"$v\", /" >> "$out"
done
