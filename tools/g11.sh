#!/bin/bash
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "acc64 or factor_matches" 2>&1 | grep -E "passed|failed|FAILED|Max abs|Mismatch" | head -30
