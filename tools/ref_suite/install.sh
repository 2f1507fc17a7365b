#!/bin/bash
# Install the UNMODIFIED reference package (citysplat, /root/reference/pkg) into
# baseline/_ref (git-ignored, travels to the GPU box with the snapshot) and
# place its own test directory beside it, so its suite can run on the B200
# through the drop-in shim (tools/ref_suite/cs_shim.py).  Needs /root/reference
# (this container only); nothing here is committed.
set -e
cd "$(dirname "$0")/../.."
rm -rf /tmp/cs_refpkg && cp -r /root/reference/pkg /tmp/cs_refpkg
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target baseline/_ref /tmp/cs_refpkg
rm -rf baseline/_ref/citysplat_tests && cp -r /root/reference/pkg/tests baseline/_ref/citysplat_tests
echo "installed: $(ls baseline/_ref)"
