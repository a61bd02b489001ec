#!/bin/bash
# Round-end evidence on one B200 (run through gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash diag/final_evidence.sh'
# GPU tests, the bench lines (240-step headline, the driver's 20-step configuration, SH degree 3,
# the reference arm, the C5 mapping loop), the ncu launch list of the timed region and the
# full-set raw export of one L2 -> L1 -> L0 cycle. Summaries: profiles/summarize.py.
out=gpurun_out
mkdir -p $out
python -m pytest tests -m gpu -x -q > $out/r2_gputest.log 2>&1
echo "tests rc=$?" >> $out/r2_gputest.log
python bench.py --steps 240 --warmup 24 > $out/r2_bench.json 2>> $out/r2_bench.err
python bench.py --steps 20 --warmup 5 > $out/r2_bench_20.json 2>> $out/r2_bench.err
python bench.py --steps 240 --warmup 24 --sh-degree 3 > $out/r2_bench_d3.json 2>> $out/r2_bench.err
python bench.py --steps 20 --warmup 5 --sh-degree 3 --no-cpu-baseline > $out/r2_bench_d3_20.json 2>> $out/r2_bench.err
timeout 400 python bench.py --impl reference > $out/r2_bench_reference.json 2>> $out/r2_bench.err
timeout 600 python bench.py --workload c5 > $out/r2_c5.json 2>> $out/r2_bench.err
# the checked build (device-side bounds assertions; build it first: diag/build_variant.sh checked -DGSB_CHECKS)
if [ -f diag/_variants/checked/libgsmap_b200.so ]; then
  (export GSMAP_B200_VARIANT=checked
   python -c "from paper_2411_02703_b200 import gsmap; print(gsmap.LIB_PATH)" > $out/r2_checked_gputest.log 2>&1
   python -m pytest tests -m gpu -q >> $out/r2_checked_gputest.log 2>&1
   echo "tests rc=$?" >> $out/r2_checked_gputest.log
   python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $out/r2_checked_bench.json 2>> $out/r2_bench.err
   echo "bench rc=$?" >> $out/r2_checked_gputest.log
   timeout 900 python bench.py --workload c5 > $out/r2_checked_c5.json 2>> $out/r2_bench.err
   echo "c5 rc=$?" >> $out/r2_checked_gputest.log)
fi
export GS_PROFILE_RANGE=1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $out/r2_launches.csv python bench.py --profile-only --steps 3 --warmup 3 --no-e2e > $out/ncu1.log 2>&1
ncu --set full --clock-control none --profile-from-start off -c 80 -o /tmp/prof_all \
    python bench.py --profile-only --steps 3 --warmup 3 --no-e2e > $out/ncu2.log 2>&1
ncu -i /tmp/prof_all.ncu-rep --page raw --csv > $out/r2_prof_all_raw.csv 2>&1
ls -la $out/r2_*
