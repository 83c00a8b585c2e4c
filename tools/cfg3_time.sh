#!/bin/bash
# config 3 (TD / QD LU n=2048 K=128, 3M and 4M) device timings via bench.py
for k in 3 4; do for m in 3m 4m; do
python bench.py --n 2048 --K 128 --k $k --method $m --steps 3 --warmup 1 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('k=$k $m', round(d['ms_per_step'],1), 'ms', round(d['value'],2), 'GFLOP/s', 'gemm frac', round(d['roofline']['frac'],3))"
done; done
