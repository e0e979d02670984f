timeout 600 python -m pytest tests -m gpu -x -q -k "resident or scene or prewalk or dropin or seeds" > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
for i in 1 2; do SEPSO_RESIDENT=1 timeout 120 python tools/e2e_fit.py; done
