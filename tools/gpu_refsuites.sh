mkdir -p gpurun_out
for t in test_container_b200 test_harness_b200; do (cd oracle/_ref && timeout 900 ./$t > ../../gpurun_out/$t.log 2>&1; echo "$t rc=$?"; tail -5 ../../gpurun_out/$t.log); done
(cd oracle/_ref && timeout 1200 ./acceptance_b200 > ../../gpurun_out/acceptance_b200.log 2>&1; echo "acceptance rc=$?"; tail -15 ../../gpurun_out/acceptance_b200.log)
timeout 900 python -m pytest tests/test_gpu_cpp_dp.py -q -x 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
