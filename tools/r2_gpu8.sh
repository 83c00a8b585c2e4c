#!/bin/bash
O=gpurun_out/r2; mkdir -p $O
python -m pytest tests -m gpu -q -x --ignore=tests/ref_suite > $O/gpu_tests_f.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests_f.log
tail -5 $O/gpu_tests_f.log
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],1), "ms", round(d["value"],1), "GFLOP/s", "frac", round(d["roofline"]["frac"],3))'
{
for mb in 4 3 2; do echo "== MPC_TDQD_MINB=$mb"; MPC_TDQD_MINB=$mb bash tools/cfg3_time.sh; done
echo -n "cfg2 default: "; python bench.py --n 4096 --K 256 --steps 5 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin 2>/dev/null | python -c "$P"
echo -n "cfg4 default: "; python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin 2>/dev/null | python -c "$P"
} > $O/defaults_f.txt 2>&1
cat $O/defaults_f.txt
bash tools/r2_sanitize.sh racecheck
