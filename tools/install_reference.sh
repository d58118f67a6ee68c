#!/bin/sh
# The one offline install of the reference (task rules): the unmodified
# `vortexfmm` package into the git-ignored baseline/_ref/ (it travels to the
# GPU box with the gpurun snapshot; nothing of it enters the repo history),
# plus its own test suite, which tests/test_reference_suite.py runs through
# the GPU evaluate (harness integration).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/vfmm_refpkg && cp -r /root/reference/pkg /tmp/vfmm_refpkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/vfmm_refpkg
rm -rf baseline/_ref/reference_tests
cp -r /root/reference/pkg/tests baseline/_ref/reference_tests
cp /root/reference/pkg/study.cfg baseline/_ref/reference_tests/study.cfg  # acceptance criterion 7 reads it
echo "installed vortexfmm into baseline/_ref"
