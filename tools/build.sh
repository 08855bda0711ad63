#!/bin/bash
# Rebuild the sm_100a library from any working directory; prints errors only
# and exits non-zero when the build fails.
cd "$(dirname "$0")/.." || exit 1
out=$(python -m paper_1502_04265_b200._build 2>&1); rc=$?
if [ $rc -ne 0 ]; then echo "$out" | grep -E "error|Error" | head -20; echo "BUILD FAILED"; exit 1; fi
ls -la --time-style=+%T paper_1502_04265_b200/libpiecy_b200.so | awk '{print "lib built", $6}'
