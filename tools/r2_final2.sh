#!/bin/bash
# final default bench line with the final library + the full suite, then the
# oracle's ill-conditioned n=8192 K=512 record on the box's host cores
O=gpurun_out/r2f; mkdir -p $O gpurun_out/r2
python -m pytest tests -m gpu -q -x > $O/gpu_tests2.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests2.log
tail -4 $O/gpu_tests2.log
python bench.py > $O/bench_cfg4_final2.json 2> $O/bench_cfg4_final2.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$O/bench_cfg4_final2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['fp64_pct_of_measured_peak'])"
timeout 2700 python oracle/gen_cfg4.py ill_n8192 --n 8192 --out gpurun_out/r2/cfg4_ill_n8192.json > gpurun_out/r2/gen_ill_n8192.log 2>&1
tail -2 gpurun_out/r2/gen_ill_n8192.log; ls -la gpurun_out/r2/cfg4_ill_n8192.json
