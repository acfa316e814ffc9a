# stem (s2d) parity + timing
timeout 600 python -m pytest tests -m gpu -x -q -k "stem" 2>&1 | tail -5
timeout 300 python scripts/stem_probe.py 256 8 --direct 2>&1 | tail -40
timeout 300 python scripts/stem_probe.py 16 4 2>&1 | tail -20
