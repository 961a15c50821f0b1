#!/bin/bash
# A/B of run-time knobs on the GPU box (dev helper): build, the named GPU
# test files, then a short bench per (workload, env variant).
# Usage: TESTS="tests/a.py -k x" WORKLOADS="lfr1m sbm100k" bash tools/gpu_ab_env.sh "A=1" "A=0 B=2" ...
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  eval timeout 1500 python -m pytest $TESTS -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "pytest=$?"; tail -5 gpurun_out/ab_pytest.log
fi
for wl in ${WORKLOADS:-lfr1m sbm100k rmat22}; do
  for v in "$@"; do
    tag=$(echo "$v" | tr ' =' '_-')
    env $v timeout 300 python bench.py --workload $wl --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/ab_${wl}_${tag}.json 2> gpurun_out/ab_${wl}_${tag}.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('RESULT', sys.argv[2], sys.argv[3], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d.get('breakdown_ms',{}).items() if k in ('potentials','ggd')})" gpurun_out/ab_${wl}_${tag}.json $wl "$v"
  done
done
