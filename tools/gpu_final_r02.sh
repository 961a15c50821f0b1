#!/bin/bash
# r02 measurement pass on the GPU box (repo root): GPU tests, smoke, bench
# (LFR / SBM / R-MAT), reference arm, launch list and ncu captures, sanitizer
# runs, end-to-end QC time, shard balance. Outputs in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench_ref=$?"
python bench.py --workload sbm100k > gpurun_out/bench_sbm.json 2> gpurun_out/bench_sbm.err; echo "bench_sbm=$?"
python bench.py --workload rmat22 --steps 10 > gpurun_out/bench_rmat.json 2> gpurun_out/bench_rmat.err; echo "bench_rmat=$?"
timeout 900 python bench.py --hop-cap 2 --steps 5 --no-e2e --cpu-seconds 6 > gpurun_out/bench_khop_lfr.json 2> gpurun_out/bench_khop_lfr.err; echo "bench_khop=$?"
bash tools/gpu_profile_r02.sh > gpurun_out/profile.log 2>&1; echo "profile=$?"
GQC_SLAB_TIMEOUT_MS=600000 timeout 1800 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck=$?"
GQC_SLAB_TIMEOUT_MS=600000 timeout 1800 compute-sanitizer --tool racecheck --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck=$?"
timeout 900 python tools/e2e_qc.py --repeat 3 > gpurun_out/e2e_qc.json 2> gpurun_out/e2e_qc.err; echo "e2e_qc=$?"
for w in rmat22 lfr1m; do timeout 300 python tools/shard_balance.py --workload $w > gpurun_out/balance_$w.json 2> gpurun_out/balance_$w.err; done
timeout 300 python tools/single_sigma_probe.py > gpurun_out/single_sigma.json 2> gpurun_out/single_sigma.err; echo "single=$?"
