#!/bin/bash
O=gpurun_out/r2; mkdir -p $O gpurun_out/r2b
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "grid_panel or implementations_agree or strassen or max_rel_err" > $O/gpu_tests_g.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests_g.log
tail -6 $O/gpu_tests_g.log
python tools/lu_breakdown.py 2048 128 blocked 3 > $O/cfg3_breakdown.txt 2>&1
python tools/lu_breakdown.py 2048 128 blocked 4 >> $O/cfg3_breakdown.txt 2>&1
MPC_TRACE=1 python tools/lu_breakdown.py 2048 128 blocked 3 2>&1 | grep TRACE | tail -17 >> $O/cfg3_breakdown.txt
cat $O/cfg3_breakdown.txt
NCU="ncu --set full --clock-control none --import-source on"
cap() {
  local name=$1 kre=$2 skip=$3 cnt=$4; shift 4
  $NCU -k regex:$kre --launch-skip $skip -c $cnt -o gpurun_out/r2b/$name "$@" > gpurun_out/r2b/ncu_$name.log 2>&1
  ncu -i gpurun_out/r2b/$name.ncu-rep --page details --csv > gpurun_out/r2b/${name}_details.csv 2>/dev/null
  ncu -i gpurun_out/r2b/$name.ncu-rep --page raw --csv > gpurun_out/r2b/${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/r2b/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/r2b/${name}_sass.csv 2>/dev/null
  gzip -f gpurun_out/r2b/${name}_sass.csv
  rm -f gpurun_out/r2b/$name.ncu-rep
}
cap panel_grid panel_grid_kernel 40 1 python tools/lu_breakdown.py 4096 256 blocked
cap gemm_td gemm_kernel 0 1 python tools/one_eft_rect.py 3 3m 1920 128 1920
cap gemm_qd gemm_kernel 0 1 python tools/one_eft_rect.py 4 3m 1920 128 1920
cap laswp laswp_kernel 200 1 python tools/lu_breakdown.py 4096 256 blocked
cap gemm_dd_lu gemm_kernel 60 1 python tools/lu_breakdown.py 8192 512 blocked
ls -la gpurun_out/r2b
