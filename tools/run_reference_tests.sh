#!/usr/bin/env bash
# Runs the reference's OWN hot-path tests (pkg/tests/test_{gridseq,skiparse,anyres,attention,ssp}.py
# and their naive oracles) unmodified against this package through the `osp` import shim in
# compat/osp, on a B200 via gpurun.  Run from the build container, where /root/reference exists:
# the test files are copied to a transient, git-ignored directory for the one call and deleted
# afterwards (they are never part of the repository).
set -u
REF=${REF:-/root/reference/pkg/tests}
cd "$(dirname "$0")/.."
rm -rf .reftests_tmp && mkdir -p .reftests_tmp
cp $REF/oracles.py $REF/test_gridseq.py $REF/test_skiparse.py $REF/test_anyres.py $REF/test_attention.py \
   $REF/test_ssp.py .reftests_tmp/
/usr/local/graft/bin/gpurun --timeout ${TIMEOUT:-900} -- \
  'mkdir -p gpurun_out/reftests; cd .reftests_tmp && PYTHONPATH=$GRAFT_REPO_ROOT/compat:$GRAFT_REPO_ROOT \
   timeout 800 python -m pytest -p no:cacheprovider -q -rf '"${PYTEST_ARGS:-}"' . \
   > $GRAFT_REPO_ROOT/gpurun_out/reftests/pytest.log 2>&1; echo "rc=$?"'
rm -rf .reftests_tmp
tail -5 gpurun_out/reftests/pytest.log
