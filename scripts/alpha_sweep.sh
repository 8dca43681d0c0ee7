#!/bin/bash
for a in 1 2 4 8 16; do
  echo "#### alpha=$a"
  ALPHA=$a NSRC=16 TRACE=0 timeout 600 python scripts/level_profile.py C2 auto 2>&1 | grep "=="
  ALPHA=$a NSRC=8 TRACE=0 timeout 900 python scripts/level_profile.py C4 auto 2>&1 | grep "=="
done
