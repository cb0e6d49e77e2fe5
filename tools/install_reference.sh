#!/bin/bash
# Install the unmodified reference (numba blowchoc) into baseline/_ref
# (git-ignored; it travels to the GPU box with the gpurun snapshot), and put
# its own test files beside it (baseline/_ref/reftests) for the integration
# test that runs them through the libbbchoc binding.  Build container only.
set -e
cd "$(dirname "$0")/.."
SRC=${1:-/root/reference}
rm -rf /tmp/refcopy && cp -r "$SRC" /tmp/refcopy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/refcopy/pkg
rm -rf baseline/_ref/reftests && cp -r /tmp/refcopy/pkg/tests baseline/_ref/reftests
echo "installed: $(ls baseline/_ref)"
