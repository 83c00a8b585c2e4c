#!/bin/bash
O=gpurun_out/r2f; mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_known_answers.py -m gpu -q -x -k "cfg4 or laswp" --durations=5 > $O/gpu_tests_cfg4.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests_cfg4.log
tail -12 $O/gpu_tests_cfg4.log
