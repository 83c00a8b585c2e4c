#!/bin/bash
# Round-2 final records: full GPU suite, default bench + reference arm,
# per-config summary, launch lists, smoke.
O=gpurun_out/r2f; mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log; tail -2 $O/smoke.log
python -m pytest tests -m gpu -q -x --durations=12 > $O/gpu_tests.log 2>&1; echo "pytest exit $?" >> $O/gpu_tests.log
tail -18 $O/gpu_tests.log
python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench exit $?"
python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
Q="--no-e2e --no-cpu --no-accuracy --no-dropin"
P='import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); a=d.get("alt_real_kernel") or {}; print(round(d["ms_per_step"],2), "ms", round(d["value"],1), d["unit"], "frac", round(d["roofline"]["frac"],3), "| alt", a.get("real_kernel"), round(a.get("ms_per_step",0),2), "ms", round(a.get("value",0),1))'
{
echo "# one B200, round 2 final (tools/r2_final.sh); alt = the other real kernel (ozaki)"
echo -n "cfg4 DD LU n=16384 K=512 3M (ill-conditioned input): "; python bench.py --ill --steps 2 --warmup 3 $Q 2>/dev/null | python -c "$P"
echo -n "cfg2 DD LU n=4096 K=256 3M: "; python bench.py --n 4096 --K 256 --steps 5 --warmup 3 $Q 2>/dev/null | python -c "$P"
echo -n "cfg2 DD LU n=4096 K=256 4M: "; python bench.py --n 4096 --K 256 --method 4m --steps 5 --warmup 3 $Q 2>/dev/null | python -c "$P"
for k in 3 4; do for m in 3m 4m; do
echo -n "cfg3 k=$k LU n=2048 K=128 $m: "; python bench.py --n 2048 --K 128 --k $k --method $m --steps 3 --warmup 3 $Q 2>/dev/null | python -c "$P"
done; done
for m in 3m 4m; do
echo -n "cfg1 DD cgemm n=1024 $m: "; python bench.py --workload gemm --method $m --steps 20 --warmup 5 $Q 2>/dev/null | python -c "$P"
done
for k in 3 4; do
echo -n "cgemm k=$k n=1024 3m: "; python bench.py --workload gemm --k $k --method 3m --steps 5 --warmup 3 $Q 2>/dev/null | python -c "$P"
done
echo -n "cfg0 DD LU n=128 K=32: "; python bench.py --n 128 --K 32 --steps 20 --warmup 5 $Q --no-alt 2>/dev/null | python -c "$P"
python tools/time_solve.py 16384 2 3m 3 2>&1 | tail -3
for tb in 16 32; do
echo -n "MPC_TRSM_BASE=$tb cfg2: "; MPC_TRSM_BASE=$tb python bench.py --n 4096 --K 256 --steps 5 --warmup 3 $Q --no-alt 2>/dev/null | python -c "$P"
echo -n "MPC_TRSM_BASE=$tb cfg4: "; MPC_TRSM_BASE=$tb python bench.py --steps 2 --warmup 3 $Q --no-alt 2>/dev/null | python -c "$P"
done
} > $O/configs_summary.txt 2>&1
cat $O/configs_summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv python bench.py --n 4096 --K 256 --steps 1 --warmup 1 $Q --no-alt > $O/ncu_launches_cfg2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches_cfg4_first1500.csv python bench.py --steps 1 --warmup 0 $Q --no-alt > $O/ncu_launches_cfg4.log 2>&1
gzip -f $O/launches_cfg2.csv $O/launches_cfg4_first1500.csv
MPC_TRACE=1 python tools/lu_breakdown.py 16384 512 blocked > $O/trace_cfg4.txt 2>&1
MPC_TRACE=1 python tools/lu_breakdown.py 4096 256 blocked > $O/trace_cfg2.txt 2>&1
ls -la $O
