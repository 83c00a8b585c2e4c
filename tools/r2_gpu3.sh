#!/bin/bash
O=gpurun_out/r2; mkdir -p $O
python -m pytest tests -m gpu -q -x --ignore=tests/ref_suite > $O/gpu_tests_b.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests_b.log
tail -8 $O/gpu_tests_b.log
python -m pytest tests/ref_suite -m gpu -q > $O/ref_suite_b.log 2>&1; echo "pytest exit $?" >> $O/ref_suite_b.log
tail -8 $O/ref_suite_b.log
bash tools/panel_ab.sh > $O/panel_ab.txt 2>&1
cat $O/panel_ab.txt
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin > $O/bench_cfg4_b.json 2>$O/bench_cfg4_b.err
python -c "import json; d=json.loads(open('$O/bench_cfg4_b.json').read().strip().splitlines()[-1]); print('cfg4', d['ms_per_step'], d['value'], d['roofline']['frac'])"
MPC_TRACE=1 python tools/lu_breakdown.py 16384 512 blocked > $O/trace_cfg4_b.txt 2>&1
tail -40 $O/trace_cfg4_b.txt
