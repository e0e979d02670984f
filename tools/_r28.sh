timeout 300 python -m pytest tests -m gpu -x -q -k "scene or prewalk or batched" 2>&1 | tail -1
for v in 1 0 1 0; do SEPSO_PREWALK_BULK=$v timeout 120 python tools/c5_time.py; done
