#!/bin/bash
# Round-2 evidence run on one B200: sustained DFMA + DSMEM bulk microbenchmarks
# with clocks logged, ncu --set full captures of the hot kernels per config, compute-sanitizer runs.
cd "$(dirname "$0")/.."
O=gpurun_out/p
mkdir -p $O
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 500 > $O/mb_smi.csv &
SMI=$!
timeout 120 ./tools/microbench/mb_dsmem 10 > $O/mb_dsmem.txt 2>&1
kill $SMI
NCU="ncu --set full --clock-control none --import-source on"
# summarise each report on the box (the .ncu-rep files are too large to bring back)
summ() {  # rep label cells
  python tools/ncu_summary.py $O/$1.ncu-rep "$2" $3 $O/$1.json "ncu --set full --clock-control none, $2" > $O/$1.summary.txt 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
  rm -f $O/$1.ncu-rep
}
timeout 400 $NCU -k regex:k_step3d --launch-skip 1 -c 1 -f -o $O/ncu_step3d_C2 python tools/profile_launch.py C2 step 1 > $O/ncu_step3d_C2.log 2>&1
summ ncu_step3d_C2 k_step3d_C2_C2 4096
timeout 500 $NCU -k regex:k_step3d --launch-skip 1 -c 1 -f -o $O/ncu_step3d_C4 python tools/profile_launch.py C4 step 1 > $O/ncu_step3d_C4.log 2>&1
summ ncu_step3d_C4 k_step3d_C4_C4 10000
timeout 300 $NCU -k regex:k_transport --launch-skip 1 -c 1 -f -o $O/ncu_transport_C4 python tools/profile_launch.py C4 transport 1 > $O/ncu_transport_C4.log 2>&1
summ ncu_transport_C4 k_transport_C4_C4 10000
timeout 300 $NCU -k regex:k_moments --launch-skip 1 -c 1 -f -o $O/ncu_moments_C2 python tools/profile_launch.py C2 moments 1 > $O/ncu_moments_C2.log 2>&1
summ ncu_moments_C2 k_moments_C2_C2 4096
timeout 300 $NCU -k regex:k_step2d --launch-skip 1 -c 1 -f -o $O/ncu_step2d_C1 python tools/profile_launch.py C1 step 1 > $O/ncu_step2d_C1.log 2>&1
summ ncu_step2d_C1 k_step2d_C1_C1 65536
for tool in memcheck racecheck synccheck; do
  for cfg in C1 C2 C4; do
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/profile_launch.py $cfg step 1 --small > $O/san_${tool}_${cfg}.txt 2>&1
    echo "exit $?" >> $O/san_${tool}_${cfg}.txt
  done
  FKS_MAX_CLUSTERS=1 timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/profile_launch.py C2 step 1 --small > $O/san_${tool}_C2_one_group.txt 2>&1
  echo "exit $?" >> $O/san_${tool}_C2_one_group.txt
done
timeout 900 $NCU -k regex:k_step3d --launch-skip 1 -c 1 -f -o $O/ncu_step3d_C5 python tools/profile_launch.py C5 step 1 > $O/ncu_step3d_C5.log 2>&1
summ ncu_step3d_C5 k_step3d_C5_C5 110592
echo done > $O/done.txt
