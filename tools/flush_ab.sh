#!/bin/bash
for lib in libsbt200_trace libsbt200_trace_dbg; do
  echo "== $lib"; SBT_LIB=$PWD/paper_1606_05696_b200/lib/$lib.so timeout 120 python tools/flush_trace.py 2>&1 | head -8
done
echo "== no flush"; SBT_TC_FLUSH=0 SBT_LIB=$PWD/paper_1606_05696_b200/lib/libsbt200_trace.so timeout 120 python tools/flush_trace.py 2>&1 | head -7
