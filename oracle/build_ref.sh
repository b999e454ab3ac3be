#!/usr/bin/env bash
# Recipe for oracle/_ref/ (git-ignored; NOT gpurun-ignored, so it travels to the GPU box):
#   _ref/site/      the UNMODIFIED reference package uhm_kit (/root/reference/pkg), installed
#                   with pip --target (a Python package: "compiled" = installed, nothing edited)
#   _ref/tests/     the reference's own test modules, run under paper_2405_15573_b200.install()
#                   by tests/test_gpu_reference_suite.py (the reference's matvec pins on the GPU)
#   _ref/operators/ real compress-path BASELINE operators built by the reference here
#                   (tools/export_ref_operator.py), with the reference's own outputs
# Test infrastructure only: the product package never imports anything under oracle/.
# Runs in the build container (where /root/reference exists); a no-op elsewhere.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${UHM_REF:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$REF/src/uhm_kit" ]; then
    echo "build_ref: reference not present ($REF); keeping $OUT as is"
    exit 0
fi
TMP="$(mktemp -d /tmp/uhm_ref_build.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"          # the build writes egg-info next to the sources: not into /root/reference
rm -rf "$OUT/site"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$OUT/site" "$TMP/pkg"
rm -rf "$OUT/site/bin"
mkdir -p "$OUT/tests"
cp "$REF"/tests/*.py "$OUT/tests/"
python - "$OUT" <<'PY'
import hashlib, json, os, sys
out = sys.argv[1]
files = {}
for root, _, names in os.walk(os.path.join(out, "site", "uhm_kit")):
    for n in sorted(names):
        if n.endswith(".py"):
            p = os.path.join(root, n)
            files[os.path.relpath(p, out)] = hashlib.sha256(open(p, "rb").read()).hexdigest()
json.dump({"source": "/root/reference/pkg", "files": files}, open(os.path.join(out, "MANIFEST.json"), "w"), indent=1)
print(f"build_ref: uhm_kit installed into {out}/site ({len(files)} modules)")
PY
