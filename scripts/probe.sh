for a in 0.25 0.5 1 2 4; do
ALPHA=$a NSRC=16 TRACE=0 timeout 300 python scripts/level_profile.py C2 auto 2>&1 | grep "==" | sed "s/^/a=$a /"
ALPHA=$a NSRC=4 TRACE=0 timeout 300 python scripts/level_profile.py C4 auto 2>&1 | grep "==" | sed "s/^/a=$a /"
done
