#!/bin/bash
# A/B of the base-panel implementations: cooperative grid kernel (default) vs
# thread-block cluster (MPC_PANEL=cluster), alone, beside a GEMM, and in the LU
for mode in grid cluster; do
  if [ $mode = cluster ]; then export MPC_PANEL=cluster; else unset MPC_PANEL; fi
  echo "== $mode"
  python tools/one_panel.py 15872 512 2 2>&1
  python tools/one_panel.py 3840 256 3 2>&1
  python tools/one_panel.py 1920 128 3 2>&1 | head -1
  python tools/panel_contention.py 2>&1 | tail -4
  python bench.py --n 4096 --K 256 --steps 5 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', round(d['ms_per_step'],1), 'ms', round(d['value'],1), 'GFLOP/s')"
done
