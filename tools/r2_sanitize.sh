#!/bin/bash
# one compute-sanitizer tool per call: bash tools/r2_sanitize.sh racecheck|synccheck|memcheck
TOOL=$1; O=gpurun_out/r2; mkdir -p $O
for mode in grid cluster launches; do
  if [ $mode = grid ]; then unset MPC_PANEL; else export MPC_PANEL=$mode; fi
  NC=3; [ $mode = grid ] || NC=2
  echo "== $TOOL MPC_PANEL=$mode" >> $O/sanitizer_$TOOL.txt
  timeout 1500 compute-sanitizer --tool $TOOL --print-limit 20 python tools/sanitize_lu.py $NC >> $O/sanitizer_$TOOL.txt 2>&1
  echo "exit $?" >> $O/sanitizer_$TOOL.txt
done
grep -E "^==|ERROR SUMMARY|RACECHECK SUMMARY|exit|n=" $O/sanitizer_$TOOL.txt
