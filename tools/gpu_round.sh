#!/bin/bash
# One GPU session: tests, smoke, benches, ncu launch lists and one full
# capture of the top kernel.  Output under gpurun_out/ (copied to profiles/
# by hand once reviewed).  Usage: tools/gpu_round.sh [tag]
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/gputests_$TAG.log 2>&1; echo "rc=$?" >> $O/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "rc=$?" >> $O/smoke_$TAG.log
for c in cfg3 cfg2 cfg5 cfg1; do
  timeout 900 python bench.py --config $c > $O/bench_${c}_$TAG.json 2> $O/bench_${c}_$TAG.err
done
timeout 600 python bench.py --impl reference > $O/bench_ref_cfg3_$TAG.json 2> $O/bench_ref_cfg3_$TAG.err
# launch lists (cold-cache, serialised: shares only) of the bench command
timeout 900 ncu --graph-profiling node --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:spmv_ -c 40 --csv --log-file $O/launches_cfg3_$TAG.csv \
  python bench.py --config cfg3 --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in cfg2:1 cfg5:1; do
  timeout 600 ncu --graph-profiling node --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:spmv_ -c 12 --csv --log-file $O/launches_${c%%:*}_$TAG.csv \
    python tools/profile_spmv.py --config ${c%%:*} --chains ${c##*:} --steps 6 > /dev/null 2>&1
done
# one full capture of the dominant kernel (first stripe pass at cfg3)
timeout 900 ncu --set full --import-source on --graph-profiling node --clock-control none -k regex:spmv_pass -s 8 -c 1 \
  -o $O/full_cfg3_$TAG python tools/profile_spmv.py --config cfg3 --chains 2 --steps 4 > /dev/null 2>&1
# dense-X projection (tensor-core digit GEMM vs lazy CUDA-core path)
for tc in 1 0; do SLD_DENSE_TC=$tc timeout 300 python tools/bench_dense.py --config cfg3 --m 2,4,8,16 --steps 48 \
  > $O/dense_cfg3_tc${tc}_$TAG.txt 2>/dev/null; done
timeout 600 ncu --set full --graph-profiling node --clock-control none -k regex:tc_digit_gemm -s 2 -c 1 \
  -o $O/full_tcgemm_$TAG python tools/bench_dense.py --config cfg3 --m 16 --steps 4 > /dev/null 2>&1
# Mksol: Horner step timing (fused vs two kernels) and the tensor-core combination kernel
timeout 900 python tools/bench_mksol.py --config cfg3 --n 8 --degree 800 --reps 5 > $O/mksol_cfg3_$TAG.txt 2>/dev/null
timeout 600 ncu --set full --clock-control none -k regex:tcl_combine -s 4 -c 1 \
  -o $O/full_tcl_$TAG python tools/bench_mksol.py --config cfg3 --n 8 --degree 8 --reps 1 > /dev/null 2>&1
# DRAM bytes per step of the benched layouts (bench.py reads profiles/traffic_*.json)
python tools/traffic_from_launches.py $O/launches_cfg3_$TAG.csv cfg3 2 4 $O/traffic_cfg3_g2_$TAG.json "spmv_pass<7, 2," > /dev/null
python tools/traffic_from_launches.py $O/launches_cfg2_$TAG.csv cfg2 1 1 $O/traffic_cfg2_g1_$TAG.json > /dev/null
python tools/traffic_from_launches.py $O/launches_cfg5_$TAG.csv cfg5 1 1 $O/traffic_cfg5_g1_$TAG.json > /dev/null
# summaries of the full captures; only the SpMV report travels back (gpurun
# copies at most 64 MiB of gpurun_out/)
for r in $O/full_cfg3_$TAG $O/full_tcgemm_$TAG $O/full_tcl_$TAG; do
  [ -f $r.ncu-rep ] && python tools/ncu_summary.py $r.ncu-rep $r.json > /dev/null 2>&1
done
rm -f $O/full_tcgemm_$TAG.ncu-rep $O/full_tcl_$TAG.ncu-rep
tail -2 $O/gputests_$TAG.log; tail -1 $O/smoke_$TAG.log
