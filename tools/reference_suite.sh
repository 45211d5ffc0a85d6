#!/bin/bash
# Run the REFERENCE's own test-suite (pkg/tests + the opentm_client bindings tests)
# against this build through the `opentm` drop-in shim (integration/opentm).
#
#   tools/reference_suite.sh stage   # here: copy the reference tests into .reftests/
#                                    # (git-ignored; travels to the GPU box with gpurun)
#   tools/reference_suite.sh run     # on the GPU box: pytest them, log to gpurun_out/
#
# The reference sources are never committed: .reftests/ is scratch for one run.
set -u
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
case "${1:-run}" in
stage)
    rm -rf "$ROOT/.reftests"
    mkdir -p "$ROOT/.reftests"
    cp -r /root/reference/pkg/tests "$ROOT/.reftests/tests"
    cp -r /root/reference/pkg/bindings/src "$ROOT/.reftests/bindings_src"
    cp -r /root/reference/pkg/bindings/tests "$ROOT/.reftests/bindings_tests"
    printf '[pytest]\nmarkers =\n    slow: long-running optimization cases\n' > "$ROOT/.reftests/pytest.ini"
    ;;
run)
    cd "$ROOT/.reftests" || exit 1
    mkdir -p "$ROOT/gpurun_out"
    PYTHONPATH="$ROOT/integration:$ROOT/.reftests/bindings_src:$ROOT" PYTHONDONTWRITEBYTECODE=1 \
        python -m pytest tests bindings_tests -q -rfEs -p no:cacheprovider --timeout 1800 \
        -o junit_family=xunit2 --junitxml="$ROOT/gpurun_out/reference_suite.xml" \
        > "$ROOT/gpurun_out/reference_suite.log" 2>&1
    echo "reference suite rc $?"
    tail -40 "$ROOT/gpurun_out/reference_suite.log"
    ;;
esac
