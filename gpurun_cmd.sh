#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout 600 python bench.py --steps 3 --warmup 3 --skip-cpu --recall-q 0 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c2', '%.3e'%j['value'], 'e2e %.3e'%j['e2e']['value'], j['e2e']['api'])"
