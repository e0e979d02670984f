timeout 120 python tools/phase_probe.py 2>&1 | sed -n 2,5p | grep -o "init: [^|]*"
timeout 120 python tools/phase_flush.py 2>&1 | tail -4 | grep -o "init: [^|]*"
