for L in lib lib_nodry lib lib_nodry; do echo "== $L"; SEPSO_LIB=paper_2308_10169_b200/$L/libsepso_cuda.so timeout 120 python tools/e2e_fit.py; done
