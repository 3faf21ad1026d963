#!/bin/bash
# Round-2 final evidence on one B200: GPU parity suite, smoke, bench lines for C1-C5 and the
# reference arm, and the ncu launch list of the default bench command.
cd "$(dirname "$0")/.."
O=gpurun_out/final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "exit $?" >> $O/smoke.log
FKS_LIB_VARIANT=checked timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_checked.log 2>&1; echo "exit $?" >> $O/pytest_gpu_checked.log
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
for cfg in C1 C3 C4 C5; do
  python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
echo done > $O/done.txt
