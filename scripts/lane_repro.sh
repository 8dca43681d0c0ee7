#!/bin/bash
# C4 lanes 4 with the given library build, fresh processes, 4 timed sets each
for i in 1 2 3 4 5 6 7 8; do timeout 100 python -u scripts/lane_sweep.py C4 4,4,4,4 2>&1 | grep -cE "lanes 4 GTEPS" ; done
