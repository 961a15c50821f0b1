#!/bin/bash
# r02 closing measurement pass on the GPU box (repo root): GPU tests, smoke,
# bench (LFR / SBM / R-MAT / k-hop), reference arm, the default command's
# launch list, ncu --set full captures of the potential, successor and label
# kernels per workload and of the K1 replay (SBM), end-to-end QC time,
# single-sigma probe, shard balance. Outputs in gpurun_out/ (tools/
# profiles_from_run.sh then refreshes profiles/).
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench_ref=$?"
python bench.py --workload sbm100k > gpurun_out/bench_sbm.json 2> gpurun_out/bench_sbm.err; echo "bench_sbm=$?"
python bench.py --workload rmat22 --steps 10 > gpurun_out/bench_rmat.json 2> gpurun_out/bench_rmat.err; echo "bench_rmat=$?"
timeout 900 python bench.py --hop-cap 2 --steps 5 --no-e2e --cpu-seconds 6 > gpurun_out/bench_khop_lfr.json 2> gpurun_out/bench_khop_lfr.err; echo "bench_khop=$?"
python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launches.log 2>&1; echo "ncu_launches=$?"
for w in lfr1m sbm100k rmat22; do
  ncu --set full --clock-control none --import-source on -k regex:"potential_warp|successors_kernel|chase_kernel|roots_kernel" -s 4 -c 4 \
      -o gpurun_out/r02_full_$w python bench.py --profile --steps 1 --warmup 1 --workload $w > gpurun_out/ncu_full_$w.log 2>&1
  echo "ncu_full_$w=$?"
done
ncu --set full --clock-control none --import-source on -k regex:"potential_warp" -s 1 -c 1 \
    -o gpurun_out/r02_full_replay_sbm100k python bench.py --profile --steps 1 --warmup 1 --workload sbm100k --kernel replay \
    > gpurun_out/ncu_full_replay.log 2>&1; echo "ncu_replay=$?"
timeout 900 python tools/e2e_qc.py --repeat 3 > gpurun_out/e2e_qc.json 2> gpurun_out/e2e_qc.err; echo "e2e_qc=$?"
timeout 300 python tools/single_sigma_probe.py > gpurun_out/single_sigma.json 2> gpurun_out/single_sigma.err; echo "single=$?"
for w in rmat22 lfr1m; do timeout 300 python tools/shard_balance.py --workload $w > gpurun_out/balance_$w.json 2> gpurun_out/balance_$w.err; done
