for flags in "-DAM_NJ4_NST=3 -DAM_NJ4_CPS=2" "-DAM_NJ4_NST=2 -DAM_NJ4_CPS=4"; do
  AM_BUILD_FLAGS="$flags" python -c "from paper_2106_10031_b200 import build; build.build(force=True)" > /dev/null 2>&1 || { echo "build failed: $flags"; continue; }
  echo "== $flags"
  timeout 600 python tools/env_ab.py --net deepsdf --max-cells 1000000 --repeat 3 "AM_GEMM_NJ4=0" "AM_GEMM_NJ4=1" 2>&1 | grep "BFS wall"
done
