for i in 1 2; do SEPSO_RESIDENT=1 timeout 120 python tools/e2e_fit.py; SEPSO_RESIDENT=0 timeout 120 python tools/e2e_fit.py; done
