#!/bin/bash
O=gpurun_out/r2; mkdir -p $O
python -m pytest tests -m gpu -q -x --ignore=tests/ref_suite > $O/gpu_tests_e.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests_e.log
tail -5 $O/gpu_tests_e.log
B="--steps 5 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],1), "ms", round(d["value"],1), "GFLOP/s", "frac", round(d["roofline"]["frac"],3))'
{
python tools/one_panel.py 15872 512 2 2>&1
python tools/one_panel.py 3840 256 3 2>&1
bash tools/cfg3_time.sh
for coop in 1 0; do
for cap in 0 260 222 148; do
  echo -n "cfg2 MPC_PANEL_COOP=$coop MPC_GEMM_CAP=$cap: "; MPC_PANEL_COOP=$coop MPC_GEMM_CAP=$cap python bench.py --n 4096 --K 256 $B 2>/dev/null | python -c "$P"
done
done
MPC_GEMM_CAP=222 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cfg2 or cfg0 or ill or lu_vs_oracle" 2>&1 | tail -2
for cap in 0 280 260 222; do
  echo -n "cfg4 plain launch MPC_GEMM_CAP=$cap: "; MPC_GEMM_CAP=$cap python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin 2>/dev/null | python -c "$P"
done
} > $O/cap_ab2.txt 2>&1
cat $O/cap_ab2.txt
MPC_GEMM_CAP=260 MPC_TRACE=1 python tools/lu_breakdown.py 16384 512 blocked 2>&1 | tail -40 > $O/trace_cfg4_cap260_plain.txt
head -8 $O/trace_cfg4_cap260_plain.txt; tail -12 $O/trace_cfg4_cap260_plain.txt
