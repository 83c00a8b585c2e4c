#!/bin/bash
# Runs oracle/gen_cfg4.py for one cfg4 input on the GPU box's 16 host cores in
# two gpurun calls (the per-call limit is 60 min; the factorization needs
# ~62): stage A leaves the matrix in /tmp on the box, stage B must land on
# the same box (gpurun reuses it when the next call follows within 5 min).
V=$1
G=/usr/local/graft/bin/gpurun
$G --timeout 3400 -- "mkdir -p gpurun_out/r2; rm -rf /tmp/cfg4_$V; python oracle/gen_cfg4.py $V --stage A --state /tmp/cfg4_$V > gpurun_out/r2/gen_cfg4_${V}_A.log 2>&1; tail -2 gpurun_out/r2/gen_cfg4_${V}_A.log; ls -la /tmp/cfg4_$V" || exit 1
$G --timeout 3400 -- "mkdir -p gpurun_out/r2; ls -la /tmp/cfg4_$V || exit 7; python oracle/gen_cfg4.py $V --stage B --state /tmp/cfg4_$V --out gpurun_out/r2/cfg4_$V.json > gpurun_out/r2/gen_cfg4_${V}_B.log 2>&1; tail -2 gpurun_out/r2/gen_cfg4_${V}_B.log; ls -la gpurun_out/r2/cfg4_$V.json; rm -rf /tmp/cfg4_$V"
