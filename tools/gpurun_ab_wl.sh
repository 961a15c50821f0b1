#!/bin/bash
# A/B on one workload: [BENCH_ARGS=...] bash tools/gpurun_ab_wl.sh <workload> "sed-expr" ... (dev helper)
set -e
wl=$1; shift
run() {
  python bench.py --profile --steps 5 --warmup 2 --workload $wl $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['breakdown_ms'])" | tee -a gpurun_out/ab.log
}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run A
for v in "$@"; do
  cp paper_2305_14641_b200/csrc/kernels.cu /tmp/k.bak
  cp paper_2305_14641_b200/csrc/ff_chain.cuh /tmp/f.bak
  cp paper_2305_14641_b200/csrc/khop.cu /tmp/h.bak
  sed -i "$v" paper_2305_14641_b200/csrc/kernels.cu paper_2305_14641_b200/csrc/ff_chain.cuh paper_2305_14641_b200/csrc/khop.cu
  make -s > /dev/null 2>&1
  run "$v"
  cp /tmp/k.bak paper_2305_14641_b200/csrc/kernels.cu
  cp /tmp/f.bak paper_2305_14641_b200/csrc/ff_chain.cuh
  cp /tmp/h.bak paper_2305_14641_b200/csrc/khop.cu
done
make -s > /dev/null 2>&1
run A2
