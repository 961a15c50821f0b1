#!/bin/bash
# A/B helper for the GPU box: build the library with a sed-edited variant and
# print the potential-kernel time of a short bench (dev helper).
set -e
run() {
  echo "== $1" >> gpurun_out/ab.log
  python bench.py --profile --steps 3 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['breakdown_ms'], d['value'])" | tee -a gpurun_out/ab.log
}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run A
for v in "$@"; do
  cp paper_2305_14641_b200/csrc/kernels.cu /tmp/k.bak
  cp paper_2305_14641_b200/csrc/ff_chain.cuh /tmp/f.bak
  sed -i "$v" paper_2305_14641_b200/csrc/kernels.cu paper_2305_14641_b200/csrc/ff_chain.cuh
  make -s > /dev/null 2>&1
  run "$v"
  cp /tmp/k.bak paper_2305_14641_b200/csrc/kernels.cu
  cp /tmp/f.bak paper_2305_14641_b200/csrc/ff_chain.cuh
done
make -s > /dev/null 2>&1
