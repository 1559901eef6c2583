#!/bin/bash
# The documented A/B switches still give bit-exact results: a subset of the GPU parity tests under each of them.
for sw in SK_PIPELINE=0 SK_FUSE_H=0 SK_TRANSPOSE_REGS=0 SK_FUSE_COLS=0 SK_NO_GRAPH=1 SK_WAVE_KERNEL=0 SK_PDL=0 SK_PANEL_REPL=0 SK_GROUP_PIPELINE=0 SK_GROUP_RESOLVER=1; do
  echo "== $sw"
  env $sw timeout 900 python -m pytest tests/test_gpu_tableau_parity.py tests/test_gpu_rows_parity.py -m gpu -q -x --timeout 600 -k "surface or d71 or random_circuits or C4 or c4 or group" 2>&1 | tail -1
done
