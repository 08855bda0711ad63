#!/bin/bash
# Rebuild the sm_100a library from any working directory; prints errors only.
cd "$(dirname "$0")/.." && python -m paper_1502_04265_b200._build 2>&1 | grep -E "error|Error" | head -20
ls -la --time-style=+%T paper_1502_04265_b200/libpiecy_b200.so | awk '{print "lib built", $6}'
