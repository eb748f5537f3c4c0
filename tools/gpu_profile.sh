#!/bin/bash
# Evidence pass on one B200 (run through gpurun from the repo root):
#   launch list of bench.py, ncu --set full of the near field and of one
#   product's far-field kernels, kernel timeline, configs, C5, GMRES, ranks.
# Every command first runs without ncu (the numbers), then under ncu.
set -u
O=gpurun_out/prof
mkdir -p $O
T="timeout 900"
$T python tools/ktrace.py --reps 7 --split > $O/ktrace.txt 2>&1
$T python tools/configs.py --reps 200 > $O/configs.txt 2>&1
$T python tools/configs.py --c5 > $O/configs_c5.txt 2>&1
$T python tools/solve_c4.py > $O/solve_c4.txt 2>&1
$T python tools/rank_time.py > $O/rank_time.txt 2>&1
$T ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  --no-c128 > $O/ncu_launches.log 2>&1
$T ncu --set full --clock-control none --import-source on -k regex:blockgemv -c 1 \
  -o $O/near python tools/prof_matvec.py --k 2 > $O/ncu_near.log 2>&1
$T ncu --set full --clock-control none --import-source on \
  -k regex:'level_tc|tgemm_tc3|fused_up|fused_down|radiation|reception|reduce|gather' -s 21 -c 21 \
  -o $O/far python tools/prof_matvec.py --k 2 > $O/ncu_far.log 2>&1
echo done
