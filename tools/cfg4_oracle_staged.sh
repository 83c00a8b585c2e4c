#!/bin/bash
# Runs oracle/gen_cfg4.py for one cfg4 input on the GPU box's 16 host cores in
# four gpurun calls (the per-call limit is 60 min; the factorization needs
# ~2 h there): each stage leaves the matrix in /tmp on the box and the next
# one must land on the same box (gpurun reuses it when the next call follows
# within 5 min).  bash tools/cfg4_oracle_staged.sh ill|uniform
V=$1
G=/usr/local/graft/bin/gpurun
S=/tmp/cfg4_$V
$G --timeout 3400 -- "mkdir -p gpurun_out/r2; rm -rf $S; python oracle/gen_cfg4.py $V --stage A --state $S > gpurun_out/r2/gen_cfg4_${V}_A.log 2>&1; tail -1 gpurun_out/r2/gen_cfg4_${V}_A.log; ls $S/rec.json" || exit 1
for st in B C; do
$G --timeout 3400 -- "mkdir -p gpurun_out/r2; ls $S/rec.json || exit 7; python oracle/gen_cfg4.py $V --stage $st --state $S > gpurun_out/r2/gen_cfg4_${V}_$st.log 2>&1; tail -1 gpurun_out/r2/gen_cfg4_${V}_$st.log" || exit 1
done
$G --timeout 3400 -- "mkdir -p gpurun_out/r2; ls $S/rec.json || exit 7; python oracle/gen_cfg4.py $V --stage D --state $S --out gpurun_out/r2/cfg4_$V.json > gpurun_out/r2/gen_cfg4_${V}_D.log 2>&1; tail -1 gpurun_out/r2/gen_cfg4_${V}_D.log; ls -la gpurun_out/r2/cfg4_$V.json; rm -rf $S"
