#!/usr/bin/env bash
# Run the reference's OWN test modules for the drop-in path against this
# implementation, through the `slabewald` module alias (tests/refcompat).
#
#   tools/run_reference_tests.sh stage   # build container: copy the reference's test
#                                        # modules into .refstage/ (git-ignored, deleted
#                                        # after the run; never committed)
#   tools/run_reference_tests.sh run     # GPU box: pytest .refstage against the drop-in
#   tools/run_reference_tests.sh clean
set -euo pipefail
cd "$(dirname "$0")/.."
STAGE=.refstage
MODULES="test_soewald2d.py test_rbse2d.py"
case "${1:-run}" in
  stage)
    rm -rf "$STAGE"; mkdir -p "$STAGE"
    for f in conftest.py oracles.py $MODULES; do cp "/root/reference/pkg/tests/$f" "$STAGE/"; done
    ;;
  run)
    test -d "$STAGE" || { echo "no $STAGE: run '$0 stage' in the build container first"; exit 2; }
    PYTHONPATH="$PWD/tests/refcompat:$PWD:$STAGE" python -m pytest -p refcompat_plugin \
      -p no:cacheprovider --rootdir "$STAGE" -c /dev/null -q -rxXfE $(for m in $MODULES; do echo "$STAGE/$m"; done)
    ;;
  clean) rm -rf "$STAGE" ;;
esac
