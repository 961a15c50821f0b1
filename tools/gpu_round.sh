#!/bin/bash
# Full measurement pass on the GPU box (run from the repo root under gpurun):
# build, GPU tests, smoke, bench (1 GPU), reference arm, ncu launch list and
# full captures of the top kernels. Outputs land in gpurun_out/.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench_ref=$?"
python bench.py --profile --steps 1 --warmup 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_launches.log 2>&1; echo "ncu_launches=$?"
ncu --set full --clock-control none --import-source on -k regex:"potential_warp|successors_kernel" -s 2 -c 2 \
    -o gpurun_out/prof_full python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
python bench.py --workload sbm100k > gpurun_out/bench_sbm.json 2> gpurun_out/bench_sbm.err; echo "bench_sbm=$?"
python bench.py --workload rmat22 --steps 10 > gpurun_out/bench_rmat.json 2> gpurun_out/bench_rmat.err; echo "bench_rmat=$?"
timeout 600 python bench.py --workload sbm100k --hop-cap 2 --steps 10 > gpurun_out/bench_khop_sbm.json 2> gpurun_out/bench_khop_sbm.err; echo "bench_khop_sbm=$?"
timeout 900 python bench.py --hop-cap 2 --steps 5 --no-e2e --cpu-seconds 6 > gpurun_out/bench_khop_lfr.json 2> gpurun_out/bench_khop_lfr.err; echo "bench_khop_lfr=$?"
ncu --set full --clock-control none --import-source on -k regex:"khop_walk|khop2_emit" -c 2 -o gpurun_out/khop_full \
    python bench.py --hop-cap 2 --profile --steps 1 --warmup 1 > gpurun_out/khop_full.log 2>&1; echo "ncu_khop=$?"
timeout 900 python tools/e2e_qc.py > gpurun_out/e2e_qc.json 2> gpurun_out/e2e_qc.err; echo "e2e_qc=$?"
