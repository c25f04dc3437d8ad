#!/bin/bash
# Round-2 evidence on one GPU: full GPU suite, smoke, per-config benches, the
# reference arm, launch lists (cold-cache, serialised: shares only) and one
# full capture of the headline's hot pass (cfg3, one chain).  Output under
# gpurun_out/ (copied to profiles/ once reviewed).  Usage: tools/gpu_round2.sh [tag]
TAG=${1:-r02d}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/gpu_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 > $O/gputests_$TAG.log 2>&1; echo "rc=$?" >> $O/gputests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "rc=$?" >> $O/smoke_$TAG.log
for c in cfg3 cfg2 cfg5 cfg1; do
  timeout 900 python bench.py --config $c > $O/bench_${c}_$TAG.json 2> $O/bench_${c}_$TAG.err
done
timeout 900 python bench.py --impl reference > $O/bench_ref_cfg3_$TAG.json 2> $O/bench_ref_cfg3_$TAG.err
# launch lists of the bench commands (DRAM bytes per launch -> traffic_*.json)
timeout 900 ncu --graph-profiling node --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:spmv_ -c 40 --csv --log-file $O/launches_cfg3_g1_$TAG.csv \
  python bench.py --config cfg3 --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in cfg2 cfg5 cfg1; do
  timeout 600 ncu --graph-profiling node --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:"spmv_|full_fixup" -c 24 --csv --log-file $O/launches_${c}_$TAG.csv \
    python tools/profile_spmv.py --config $c --steps 8 > /dev/null 2>&1
done
python tools/traffic_from_launches.py $O/launches_cfg3_g1_$TAG.csv cfg3 1 2 $O/traffic_cfg3_g1_$TAG.json "spmv_pass<7, 1," > /dev/null
# one full capture of the hot (first) stripe pass of the headline layout
timeout 900 ncu --set full --import-source on --graph-profiling node --clock-control none -k regex:spmv_pass -s 6 -c 1 \
  -o $O/full_cfg3_g1_$TAG python tools/profile_spmv.py --config cfg3 --chains 1 --steps 4 > /dev/null 2>&1
[ -f $O/full_cfg3_g1_$TAG.ncu-rep ] && python tools/ncu_summary.py $O/full_cfg3_g1_$TAG.ncu-rep $O/ncu_cfg3_g1_$TAG.json > /dev/null 2>&1
# memcheck over the randomised chains: compute-sanitizer has since been
# closed on this pool (runs under it left GPUs needing a reset), so it is
# attempted only when SLD_MEMCHECK=1
if [ "${SLD_MEMCHECK:-0}" = 1 ]; then
  timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_stress_gpu.py -x -q \
    -k "fresh or random_chains_vs_oracle[0] or random_chains_vs_oracle[1]" > $O/memcheck_stress_$TAG.txt 2>&1
  echo "rc=$?" >> $O/memcheck_stress_$TAG.txt
fi
tail -2 $O/gputests_$TAG.log; tail -1 $O/smoke_$TAG.log
for c in cfg3 cfg2 cfg5 cfg1; do python -c "
import json; d=json.load(open('$O/bench_${c}_$TAG.json')); print('$c', round(d['value'],1), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', round(d['e2e']['value'],1))"; done
