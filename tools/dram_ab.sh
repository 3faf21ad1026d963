for v in nb4 nb5 nb6; do
  FKS_LIB_VARIANT=$v python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pl_$v.log 2>&1 && FKS_LIB_VARIANT=$v ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_step3d -s 3 -c 1 --csv --log-file gpurun_out/dram_$v.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
