#!/bin/bash
# A/B of an arbitrary command over sed-edited builds (dev helper):
#   bash tools/gpurun_ab_cmd.sh "<command>" "sed-expr" ...
set -e
cmd=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== A: $(eval $cmd 2>/dev/null | tail -1)" | tee -a gpurun_out/ab.log
for v in "$@"; do
  for f in kernels.cu ff_chain.cuh khop.cu capi.cu; do cp paper_2305_14641_b200/csrc/$f /tmp/$f.bak; done
  sed -i "$v" paper_2305_14641_b200/csrc/kernels.cu paper_2305_14641_b200/csrc/ff_chain.cuh \
      paper_2305_14641_b200/csrc/khop.cu paper_2305_14641_b200/csrc/capi.cu
  make -s > /dev/null 2>&1
  echo "== $v: $(eval $cmd 2>/dev/null | tail -1)" | tee -a gpurun_out/ab.log
  for f in kernels.cu ff_chain.cuh khop.cu capi.cu; do cp /tmp/$f.bak paper_2305_14641_b200/csrc/$f; done
done
make -s > /dev/null 2>&1
