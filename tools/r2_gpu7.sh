#!/bin/bash
O=gpurun_out/r2; mkdir -p $O
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],1), "ms", round(d["value"],1), "GFLOP/s", "frac", round(d["roofline"]["frac"],3))'
{
for cap in 234 222 200; do
  echo -n "cfg4 TPR=1 MPC_GEMM_CAP=$cap: "; MPC_PANEL_TPR=1 MPC_GEMM_CAP=$cap python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin 2>/dev/null | python -c "$P"
done
MPC_PANEL_TPR=1 MPC_GEMM_CAP=222 MPC_TRACE=1 python tools/lu_breakdown.py 16384 512 blocked 2>&1 | tail -40 | head -12
echo "== cfg2 trace cap 0"
MPC_TRACE=1 python tools/lu_breakdown.py 4096 256 blocked 2>&1 | tail -24
echo "== cfg2 trace cap 260"
MPC_GEMM_CAP=260 MPC_TRACE=1 python tools/lu_breakdown.py 4096 256 blocked 2>&1 | tail -24
} > $O/cap_ab3.txt 2>&1
cat $O/cap_ab3.txt
