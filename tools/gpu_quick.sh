#!/bin/bash
# Quick GPU pass for a change under development: build, the named GPU test
# files, then optional bench commands (each under its own timeout).
# Usage: bash tools/gpu_quick.sh "tests/a.py tests/b.py [-k 'expr']" "bench args 1" "bench args 2" ...
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
tests="$1"; shift
if [ -n "$tests" ]; then
  eval timeout 1200 python -m pytest $tests -m gpu -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest=$?"
  tail -15 gpurun_out/pytest_quick.log
fi
k=0
for a in "$@"; do
  k=$((k+1))
  timeout 600 python bench.py $a > gpurun_out/quick_bench_$k.json 2> gpurun_out/quick_bench_$k.err; echo "bench[$a]=$?"
  tail -c 1500 gpurun_out/quick_bench_$k.json; tail -5 gpurun_out/quick_bench_$k.err
done
