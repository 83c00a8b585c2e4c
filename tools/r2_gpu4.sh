#!/bin/bash
O=gpurun_out/r2; mkdir -p $O
python -m pytest tests -m gpu -q --ignore=tests/ref_suite > $O/gpu_tests_c.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests_c.log
tail -12 $O/gpu_tests_c.log
python -m pytest tests/ref_suite -m gpu -q > $O/ref_suite_c.log 2>&1; echo "pytest exit $?" >> $O/ref_suite_c.log
tail -8 $O/ref_suite_c.log
bash tools/cfg3_time.sh > $O/cfg3_c.txt 2>&1; cat $O/cfg3_c.txt
python tools/one_panel.py 15872 512 2 2>&1 | head -3
python tools/one_panel.py 3840 256 3 2>&1 | head -3
python bench.py --n 4096 --K 256 --steps 5 --warmup 3 --no-e2e --no-cpu --no-alt --no-accuracy --no-dropin 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', round(d['ms_per_step'],1), 'ms', round(d['value'],1), 'GFLOP/s')"
