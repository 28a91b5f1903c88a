#!/bin/bash
# Re-run the reference's test suite against the drop-in.
#   here:        tools/refsuite/run.sh stage    (copies /root/reference's package + tests into .reftest/)
#   on the box:  tools/refsuite/run.sh run TAG  (pytest per file into gpurun_out/refsuite_TAG_*.log)
set -u
cd "$(dirname "$0")/../.."
case "${1:-}" in
  stage)
    rm -rf .reftest && mkdir -p .reftest
    cp -r /root/reference/pkg/src/pactkit .reftest/pactkit
    cp /root/reference/pkg/tests/test_*.py .reftest/
    cp tools/refsuite/conftest.py .reftest/conftest.py
    ls .reftest ;;
  run)
    TAG=${2:-r02}
    cd .reftest
    for f in test_geometry test_forward test_recon test_bench test_kernels test_cli test_acceptance; do
      timeout 1200 python -m pytest $f.py -q -rfE -p no:cacheprovider --timeout 900 > ../gpurun_out/refsuite_${TAG}_$f.log 2>&1
      echo "$f: $(tail -1 ../gpurun_out/refsuite_${TAG}_$f.log)"
    done ;;
  *) echo "usage: $0 stage | run TAG"; exit 2 ;;
esac
