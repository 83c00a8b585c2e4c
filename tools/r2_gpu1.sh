#!/bin/bash
# Round-2 GPU call 1: full GPU suite (incl. the reference's API suites), the
# default bench line (cfg4) and the reference arm.
O=gpurun_out/r2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit --format=csv > $O/gpu.txt
nproc >> $O/gpu.txt; lscpu | head -20 >> $O/gpu.txt
python -m pytest tests -m gpu -q -x --durations=15 > $O/gpu_tests.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests.log
tail -30 $O/gpu_tests.log
python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench exit $?"
tail -c 3000 $O/bench_cfg4.json
python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref exit $?"
cat $O/bench_ref.json
