#!/bin/bash
export BENCH_ALLOW_SHORT=1
timeout -s KILL 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | tee gpurun_out/pytest.log
timeout 300 python bench.py --config c1 --steps 3 --warmup 3 --skip-cpu --recall-q 50 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('c1', j['value'], j['qps'], j['roofline']['frac'], {k:(v['cand_per_s']) for k,v in j['sweep'].items()})"
timeout 900 python bench.py --steps 3 --warmup 3 --skip-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; echo rc=$?
python -c "import json; j=json.load(open('gpurun_out/bench_c2.json')); print('c2', j['value'], j['qps'], j['roofline']['frac'], {k:(v['cand_per_s']) for k,v in j['sweep'].items()}, 'e2e', j['e2e']['value'])"
