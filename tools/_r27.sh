for L in lib_base lib lib_base lib; do echo "== $L"; SEPSO_LIB=paper_2308_10169_b200/$L/libsepso_cuda.so timeout 120 python tools/e2e_fit.py; done
