#!/bin/bash
# The reference's own pipeline tests against the B200 drop-in (tools/ref_shim/plugin.py).
#   bash tools/run_reference_tests.sh stage   # here: copy the unmodified reference into baseline/_ref (git-ignored)
#   bash tools/run_reference_tests.sh run     # on the GPU box (baseline/_ref travels with the snapshot)

cd "$(dirname "$0")/.."
case "${1:-run}" in
  stage)
    rm -rf baseline/_ref/src baseline/_ref/tests
    mkdir -p baseline/_ref/src
    cp -r /root/reference/pkg/src/gradcomp baseline/_ref/src/
    cp -r /root/reference/pkg/tests baseline/_ref/tests
    echo "staged reference sources + tests under baseline/_ref" ;;
  run)
    out=${2:-gpurun_out/ref_tests.log}
    PYTHONPATH=baseline/_ref/src:. python -m pytest -p tools.ref_shim.plugin -p no:cacheprovider -o addopts="" \
      --rootdir baseline/_ref -q -rA \
      baseline/_ref/tests/test_pipelines.py \
      "baseline/_ref/tests/test_acceptance.py::test_c2_collective_correctness" \
      "baseline/_ref/tests/test_acceptance.py::test_c3_transform_suite" \
      "baseline/_ref/tests/test_acceptance.py::test_c6_saturation_trend" \
      "baseline/_ref/tests/test_acceptance.py::test_c7_powersgd_properties" > "$out" 2>&1
    echo "rc=$?" >> "$out" ;;
  run-core)
    out=${2:-gpurun_out/ref_tests_core.log}
    PYTHONPATH=baseline/_ref/src:. python -m pytest -p tools.ref_shim.core_plugin -p no:cacheprovider -o addopts="" \
      --rootdir baseline/_ref -q -rA \
      baseline/_ref/tests/test_pipelines.py \
      "baseline/_ref/tests/test_acceptance.py::test_c4_quantizer_unbiasedness" \
      "baseline/_ref/tests/test_acceptance.py::test_c6_saturation_trend" > "$out" 2>&1
    echo "rc=$?" >> "$out" ;;
esac
