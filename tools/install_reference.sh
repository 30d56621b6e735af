#!/bin/bash
# Installs the unmodified reference (tntz, pure numpy) into the git-ignored
# baseline/_ref/ together with its own test suite, from a /tmp copy (the
# build writes into the source tree; /root/reference is read-only).  gpurun
# ships baseline/_ref to the GPU box, where bench.py --impl reference runs it
# and tests/test_tntz_shim.py runs its hot-path tests against the GPU.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/tntz_pkg baseline/_ref
cp -r /root/reference/pkg /tmp/tntz_pkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/tntz_pkg
cp -r /root/reference/pkg/tests baseline/_ref/tests
echo "installed: $(ls baseline/_ref)"
