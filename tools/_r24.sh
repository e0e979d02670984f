timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for L in lib_base lib lib_base lib; do echo "== $L"; SEPSO_LIB=paper_2308_10169_b200/$L/libsepso_cuda.so timeout 120 python tools/c5_time.py; SEPSO_LIB=paper_2308_10169_b200/$L/libsepso_cuda.so timeout 120 python tools/configs13.py 2>&1 | tail -3; done
