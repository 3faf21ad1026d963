#!/bin/bash
# Round-2 closing evidence after the k_step3d register-allocation change: bench lines for C1-C5 and
# the reference arm, the ncu launch list of the default command, and one ncu --set full capture of
# k_step3d on C2 (summarised on the box).
cd "$(dirname "$0")/.."
O=gpurun_out/final3
mkdir -p $O
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for cfg in C1 C3 C4 C5; do
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step3d --launch-skip 1 -c 1 -f \
    -o $O/ncu_step3d_C2 python tools/profile_launch.py C2 step 1 > $O/ncu_step3d_C2.log 2>&1
python tools/ncu_summary.py $O/ncu_step3d_C2.ncu-rep k_step3d_C2 4096 $O/ncu_step3d_C2.json \
    "ncu --set full --clock-control none, k_step3d C2 (register-usage-level 6 build)" > $O/ncu_step3d_C2.summary.txt 2>&1
rm -f $O/ncu_step3d_C2.ncu-rep
echo done > $O/done.txt
