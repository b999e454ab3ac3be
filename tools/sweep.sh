#!/bin/bash
# quick perf sweep on the GPU box: prints ms/step and roofline frac per setting
mkdir -p gpurun_out
run() {  # label, env..., args...
  local label=$1; shift
  env "$@" > /dev/null
  out=$(env $ENVV timeout 300 python bench.py $ARGS --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1)
  echo "$label $(python -c "import json,sys; d=json.loads(sys.argv[1]); print('%.4f ms frac %.3f e2e %.1f' % (d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']))" "$out" 2>/dev/null || echo "FAIL: $out" | tail -c 600)"
}
