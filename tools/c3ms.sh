#!/bin/bash
# C3 per-op milliseconds (bench_configs.py --configs 3), one line; env vars pass through.
python bench_configs.py --configs 3 --tag x 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read())['C3']['per_op']; print({k:round(v['ms'],3) for k,v in d.items()})"
