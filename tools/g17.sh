#!/bin/bash
for g in 8 0; do
  if [ $g = 0 ]; then export SBT_TC_FLUSH=0; else export SBT_TC_FLUSH_G=$g; fi
  echo "== G=$g"; timeout 300 python tools/hooi_trace.py 2>&1 | grep -v Warn | tail -45
done
