#!/usr/bin/env bash
# Install the UNMODIFIED reference package (wedgegraph 0.1.0) into the
# git-ignored baseline/_ref (it travels to the GPU box with gpurun):
#   * the package itself, built by its own setup.py (Cython _kernels -> the
#     "native" backend), offline from /opt/wheelhouse;
#   * its own test suite (pkg/tests), which tests/test_gpu_reference_suites.py
#     runs with the B200 backend injected through the reference's seam.
# Needs /root/reference (this container only).  Idempotent.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REF:-/root/reference}"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF/pkg" "$TMP/pkg"          # the build writes into the source tree
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg" >/dev/null
cp -r "$REF/pkg/tests" "$HERE/_ref/tests"
PYTHONPATH="$HERE/_ref" python -c "import wedgegraph.kernels as k; assert 'native' in k.available_backends(), k.available_backends(); print('baseline/_ref:', k.available_backends())"
