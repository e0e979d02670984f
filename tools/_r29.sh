timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for L in lib_base lib lib_base lib; do SEPSO_LIB=/root/repo/paper_2308_10169_b200/$L/libsepso_cuda.so timeout 300 python tools/c4_iters.py; done
