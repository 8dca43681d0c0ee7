#!/bin/bash
# A/B the libdawn variants given as args on C2 and C4 (level_profile summaries only)
for lib in "$@"; do
  echo "#### $lib"
  DAWN_LIB=paper_2208_04514_b200/$lib.so NSRC=16 TRACE=0 timeout 600 python scripts/level_profile.py C2 auto 2>&1 | grep "=="
  DAWN_LIB=paper_2208_04514_b200/$lib.so NSRC=6 TRACE=0 timeout 900 python scripts/level_profile.py C4 auto 2>&1 | grep "=="
done
