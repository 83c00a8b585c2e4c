#!/bin/bash
# Round-2 GPU call 2: the repo's GPU suite, the reference's API suites, the
# panel A/B timings and the ncu captures of the kernels VERDICT r1 listed.
O=gpurun_out/r2; mkdir -p $O
python -m pytest tests -m gpu -q -x --ignore=tests/ref_suite --durations=15 > $O/gpu_tests.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests.log
tail -25 $O/gpu_tests.log
python -m pytest tests/ref_suite -m gpu -q > $O/ref_suite.log 2>&1; echo "pytest exit $?" >> $O/ref_suite.log
tail -25 $O/ref_suite.log
python tools/one_panel.py 15872 512 2 > $O/panel_alone.txt 2>&1
python tools/one_panel.py 3840 256 3 >> $O/panel_alone.txt 2>&1
python tools/panel_contention.py >> $O/panel_alone.txt 2>&1
cat $O/panel_alone.txt
bash tools/prof_r2a.sh > $O/prof_r2a.log 2>&1
tail -5 $O/prof_r2a.log
