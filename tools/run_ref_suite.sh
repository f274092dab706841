#!/bin/bash
# Run the reference's own pkg/tests against the b200 backend (GPU box).
# Prerequisite (in the build container, where /root/reference exists): the
# reference installed into the git-ignored baseline/_ref, plus its tests:
#   python -m pip install --no-index --no-build-isolation --no-deps \
#       --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>
#   cp -r /root/reference/pkg/tests baseline/_ref/tests
set -e
cd "$(dirname "$0")/.."
PYTHONPATH=baseline/_ref:. PYTHONDONTWRITEBYTECODE=1 python -m pytest -p tools.ref_suite_b200 \
  -p no:cacheprovider --rootdir baseline/_ref -q -rfE baseline/_ref/tests "$@"
