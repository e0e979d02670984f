#!/bin/bash
# A/B of library builds on one box: tools/ab.sh lib lib_x lib_y ... (flush_probe per build)
for L in "$@"; do
  echo "== $L"
  SEPSO_LIB=paper_2308_10169_b200/$L/libsepso_cuda.so python tools/flush_probe.py 2>&1 | tail -2
done
