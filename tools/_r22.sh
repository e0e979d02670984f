timeout 300 python -m pytest tests -m gpu -x -q -k "resident or scene or prewalk or dropin or seeds" 2>&1 | tail -1
for L in lib lib_p4 lib_rel lib lib_p4 lib_rel; do echo "== $L"; SEPSO_LIB=paper_2308_10169_b200/$L/libsepso_cuda.so timeout 120 python tools/e2e_fit.py; done
