#!/bin/bash
# ncu --set full of the headline kernel: the step-0 trailing update of the
# cfg4 LU (gemm_kernel<2, MODE_G3, 32x32>, 15872 x 512 x 15360)
O=gpurun_out/r2c; mkdir -p $O
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<.int.2, .int.1, .int.32" --launch-skip 1 -c 1 -o $O/gemm_g3_cfg4 python tools/lu_breakdown.py 16384 512 blocked > $O/ncu_gemm_g3_cfg4.log 2>&1
ncu -i $O/gemm_g3_cfg4.ncu-rep --page details --csv > $O/gemm_g3_cfg4_details.csv 2>/dev/null
ncu -i $O/gemm_g3_cfg4.ncu-rep --page raw --csv > $O/gemm_g3_cfg4_raw.csv 2>/dev/null
rm -f $O/gemm_g3_cfg4.ncu-rep
tail -3 $O/ncu_gemm_g3_cfg4.log; ls -la $O
