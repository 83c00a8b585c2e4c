#!/bin/bash
# Round-2 ncu captures of the kernels VERDICT r1 listed as unprofiled.
# Run on the GPU box from the repo root; outputs under gpurun_out/r2a/
# (CSV exports; the .ncu-rep files are deleted to stay under the 64 MiB
# pull limit unless KEEP_REP=1).
set -x
O=gpurun_out/r2a; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
cap() {  # name, kernel regex, skip, count, command...
  local name=$1 kre=$2 skip=$3 cnt=$4; shift 4
  $NCU -k regex:$kre --launch-skip $skip -c $cnt -o $O/$name "$@" > $O/ncu_$name.log 2>&1
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page source --csv --print-source sass > $O/${name}_sass.csv 2>/dev/null
  gzip -f $O/${name}_sass.csv
  [ -n "$KEEP_REP" ] || rm -f $O/$name.ncu-rep
}
python tools/lu_breakdown.py 4096 256 blocked > $O/cfg2_breakdown.txt 2>&1
cap panel_cluster panel_cluster_kernel 40 1 python tools/lu_breakdown.py 4096 256 blocked
cap laswp laswp_kernel 200 2 python tools/lu_breakdown.py 4096 256 blocked
cap trsm_diag trsm_diag_kernel 100 1 python tools/lu_breakdown.py 4096 256 blocked
cap gemm_td gemm_kernel 0 1 python tools/one_eft_rect.py 3 3m 1920 128 1920
cap gemm_qd gemm_kernel 0 1 python tools/one_eft_rect.py 4 3m 1920 128 1920
cap ozaki_tc ozaki_tc_kernel 0 1 python tools/one_ozaki_rect.py 2 3m 8192 512
cap trsv_fwd trsv_block_kernel 200 1 python tools/time_solve.py 16384 2 3m 1
cap trsv_bwd trsv_block_kernel 700 1 python tools/time_solve.py 16384 2 3m 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python tools/lu_breakdown.py 4096 256 blocked > $O/ncu_launches.log 2>&1
ls -la $O
