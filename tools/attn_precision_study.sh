#!/bin/bash
# Fixture parity (bf16) under each K5 precision setting: bit0 = Q hi/lo, bit1 = P hi/lo.
for f in 3 2 1 0; do
  echo "== CHOREO_ATTN_FLAGS=$f"
  CHOREO_ATTN_FLAGS=$f python -m pytest tests/test_gpu_engine.py -m gpu -q -k "bf16" 2>&1 | tail -3
done
