#!/bin/bash
# A/B of compile-time variants (AM_BUILD_FLAGS) on one box: rebuild, then time configs[1]'s BFS.
#   bash tools/build_ab.sh "" "-DAM_NARROW_NSB=6 -DAM_NARROW_NACT=1" ...
for flags in "$@"; do
  AM_BUILD_FLAGS="$flags" python -c "from paper_2106_10031_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  echo "== flags: [$flags]"
  python tools/env_ab.py --repeat 10 ${AB_VARIANT:-"AM_PREFIX=1"} 2>&1 | tail -1
done
AM_BUILD_FLAGS="" python -c "from paper_2106_10031_b200 import build; build.build(force=True)" > /dev/null 2>&1
