#!/bin/bash
# quick perf sweep on the GPU box: prints ms/step, roofline frac, launch geometry and (with
# UHMV_PROFILE=1) the bulk engine's cycle accounting, one line per setting
mkdir -p gpurun_out
run() {  # label; uses $ENVV and $ARGS
  local label=$1; shift
  out=$(env $ENVV timeout 300 python bench.py $ARGS --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1)
  echo "$label $(python - "$out" <<'PY' 2>/dev/null || echo "FAIL: $(echo "$out" | tail -c 400)"
import json, sys
d = json.loads(sys.argv[1])
s = '%.4f ms frac %.3f e2e %.1f' % (d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])
L = d.get('launch') or {}
s += ' grid %s st %s smem %s' % (L.get('grid'), L.get('stages'), L.get('smem_bytes'))
c = d.get('engine_cycles')
if c:
    ks = c['kinds']
    tot = sum(v['wait_data'] + v['wait_dep'] + v['compute'] + v['overhead'] for v in ks.values())
    s += ' | prod stage %.2f slot %.2f' % (c['p_wait_stage'] / tot, c['p_wait_slot'] / tot)
    for name, v in ks.items():
        t = v['wait_data'] + v['wait_dep'] + v['compute'] + v['overhead']
        s += ' | %s %.2f: data %.2f dep %.2f comp %.2f ovh %.2f cyc/op %.0f' % (
            name, t / tot, v['wait_data'] / t, v['wait_dep'] / t, v['compute'] / t, v['overhead'] / t,
            t / max(v['ops'], 1) / (d['launch']['grid'] and 1))
print(s)
PY
)"
}
