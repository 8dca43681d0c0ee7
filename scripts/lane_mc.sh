#!/bin/bash
timeout 1200 compute-sanitizer --tool memcheck --print-limit 5 python -u scripts/lane_check.py C4 3 64 2 2>&1 | tail -40
