#!/bin/bash
export SBT_LIB=$PWD/paper_1606_05696_b200/lib/libsbt200_trace.so
echo "== FLUSH G=8"; timeout 120 python tools/flush_trace.py
echo "== FLUSH G=1"; SBT_TC_FLUSH_G=1 timeout 120 python tools/flush_trace.py
echo "== no flush"; SBT_TC_FLUSH=0 timeout 120 python tools/flush_trace.py
