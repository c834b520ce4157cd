#!/bin/bash
# Install the UNMODIFIED reference (tabserve) into baseline/_ref (git-ignored,
# shipped to the GPU box by gpurun) for the reference-caller tests
# (tests/test_reference_callers.py) and tools/cold_start.py.  The build writes
# into its source tree, so it installs from a copy; dependencies (numpy, scipy,
# cryptography) are already in the image, hence --no-deps.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/tabserve_src baseline/_ref
cp -r /root/reference /tmp/tabserve_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/tabserve_src/pkg
