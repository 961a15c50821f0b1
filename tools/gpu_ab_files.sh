#!/bin/bash
# A/B of whole-file variants on the GPU box (dev helper): bench the working
# tree, then for each ALT (a path under .ab/ holding an alternative of
# kernels.cu) swap it in, rebuild libgqc, bench; repeat the pair REPS times.
# Usage: WORKLOADS="lfr1m rmat22" REPS=2 bash tools/gpu_ab_files.sh .ab/kernels_head.cu
set -x
bench() {
  for wl in ${WORKLOADS:-lfr1m sbm100k rmat22}; do
    timeout 300 python bench.py --workload $wl --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/abf.json 2> gpurun_out/abf.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/abf.json').read().strip().splitlines()[-1]); print('RESULT', sys.argv[1], sys.argv[2], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('breakdown_ms',{}).items() if k in ('potentials','ggd')})" "$1" $wl
  done
}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
cp paper_2305_14641_b200/csrc/kernels.cu /tmp/k_work.cu
for r in $(seq ${REPS:-1}); do
  cp /tmp/k_work.cu paper_2305_14641_b200/csrc/kernels.cu; make -s paper_2305_14641_b200/libgqc.so > /dev/null 2>&1
  bench work
  for alt in "$@"; do
    cp "$alt" paper_2305_14641_b200/csrc/kernels.cu; make -s paper_2305_14641_b200/libgqc.so > /dev/null 2>&1 || echo "build failed: $alt"
    bench "$alt"
  done
done
cp /tmp/k_work.cu paper_2305_14641_b200/csrc/kernels.cu; make -s paper_2305_14641_b200/libgqc.so > /dev/null 2>&1
