#!/bin/bash
# r02 profile pass (GPU box, repo root): launch list of the default bench
# command, ncu --set full captures of the potential + successor kernels per
# workload (LFR 1M, SBM 100k, R-MAT 22) and of the K1 dense replay (SBM).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launches.log 2>&1; echo "ncu_launches=$?"
for w in lfr1m sbm100k rmat22; do
  ncu --set full --clock-control none --import-source on -k regex:"potential_warp|successors_kernel" -s 2 -c 2 \
      -o gpurun_out/r02_full_$w python bench.py --profile --steps 1 --warmup 1 --workload $w > gpurun_out/ncu_full_$w.log 2>&1
  echo "ncu_full_$w=$?"
done
ncu --set full --clock-control none --import-source on -k regex:"potential_warp" -s 1 -c 1 \
    -o gpurun_out/r02_full_replay_sbm100k python bench.py --profile --steps 1 --warmup 1 --workload sbm100k --kernel replay \
    > gpurun_out/ncu_full_replay.log 2>&1; echo "ncu_replay=$?"
