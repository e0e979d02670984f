for i in 1 2; do
timeout 60 python tools/c5_time.py 2>&1 | tail -1
SEPSO_NO_RING=1 timeout 60 python tools/c5_time.py 2>&1 | tail -1
done
SEPSO_NO_RING=1 timeout 120 python tools/phase_batch.py 2>&1 | head -1 | cut -c1-400
