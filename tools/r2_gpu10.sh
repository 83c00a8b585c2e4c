#!/bin/bash
O=gpurun_out/r2; mkdir -p $O
python -m pytest tests -m gpu -q -x --ignore=tests/ref_suite > $O/gpu_tests_h.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests_h.log
tail -5 $O/gpu_tests_h.log
python -m pytest tests/ref_suite -m gpu -q > $O/ref_suite_h.log 2>&1; echo "pytest exit $?" >> $O/ref_suite_h.log
tail -3 $O/ref_suite_h.log
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],1), "ms", round(d["value"],1), "GFLOP/s", "frac", round(d["roofline"]["frac"],3))'
{
for cap in auto 0; do
  if [ $cap = auto ]; then unset MPC_GEMM_CAP; else export MPC_GEMM_CAP=$cap; fi
  echo "== MPC_GEMM_CAP=$cap"; bash tools/cfg3_time.sh
done
unset MPC_GEMM_CAP
echo -n "cfg2 default: "; python bench.py --n 4096 --K 256 --steps 5 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin 2>/dev/null | python -c "$P"
for n in 256 192 144 128 96 64 48; do MPC_INT8_PEAK_N=$n python tools/probe_int8_n.py; done
} > $O/defaults_h.txt 2>&1
cat $O/defaults_h.txt
