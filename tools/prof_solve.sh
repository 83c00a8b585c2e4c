#!/bin/bash
# ncu of the solve kernels (n=16384 DD): CSV exports under gpurun_out/solve/
O=gpurun_out/solve; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
cap() {
  local name=$1 kre=$2 skip=$3 cnt=$4; shift 4
  $NCU -k regex:$kre --launch-skip $skip -c $cnt -o $O/$name "$@" > $O/ncu_$name.log 2>&1
  ncu -i $O/$name.ncu-rep --page details --csv > $O/${name}_details.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page raw --csv > $O/${name}_raw.csv 2>/dev/null
  ncu -i $O/$name.ncu-rep --page source --csv --print-source sass > $O/${name}_sass.csv 2>/dev/null
  gzip -f $O/${name}_sass.csv
  rm -f $O/$name.ncu-rep
}
cap trsv_fwd trsv_block_kernel 200 1 python tools/time_solve.py 16384 2 3m 1
cap trsv_bwd trsv_block_kernel 700 1 python tools/time_solve.py 16384 2 3m 1
cap perm perm_ 0 2 python tools/time_solve.py 16384 2 3m 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/time_solve.py 16384 2 3m 1 > $O/ncu_launches.log 2>&1
ls -la $O
