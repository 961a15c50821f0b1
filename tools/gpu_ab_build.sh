#!/bin/bash
# A/B of compile-time variants on the GPU box (dev helper): build, optional GPU
# tests (TESTS), short benches per workload (WORKLOADS), then for each sed
# expression: edit kernels.cu / ff_chain.cuh, rebuild libgqc, bench again.
# Usage: TESTS="tests/a.py" WORKLOADS="lfr1m" bash tools/gpu_ab_build.sh 's/A/B/' ...
set -x
bench() {
  for wl in ${WORKLOADS:-lfr1m sbm100k rmat22}; do
    timeout 300 python bench.py --workload $wl --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/abb.json 2> gpurun_out/abb.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/abb.json').read().strip().splitlines()[-1]); print('RESULT', sys.argv[1], sys.argv[2], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('breakdown_ms',{}).items() if k in ('potentials','ggd')})" "$1" $wl
  done
}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  eval timeout 1500 python -m pytest $TESTS -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest=$?"; tail -5 gpurun_out/ab_pytest.log
fi
bench default
for v in "$@"; do
  cp paper_2305_14641_b200/csrc/kernels.cu /tmp/k.bak; cp paper_2305_14641_b200/csrc/ff_chain.cuh /tmp/f.bak
  sed -i "$v" paper_2305_14641_b200/csrc/kernels.cu paper_2305_14641_b200/csrc/ff_chain.cuh
  make -s paper_2305_14641_b200/libgqc.so > /dev/null 2>&1 || echo "build failed: $v"
  bench "$v"
  cp /tmp/k.bak paper_2305_14641_b200/csrc/kernels.cu; cp /tmp/f.bak paper_2305_14641_b200/csrc/ff_chain.cuh
done
make -s paper_2305_14641_b200/libgqc.so > /dev/null 2>&1
