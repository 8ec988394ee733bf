timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_gpu_reference_suites.py::test_reference_acceptance_through_b200 > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
