# the whole GPU suite (as the driver runs it) + smoke, then the round measurement pass
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/full_suite.log 2>&1; echo suite rc=$?; tail -3 gpurun_out/full_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
bash scripts/gpu_round2_measure.sh > gpurun_out/r2m.log 2>&1; echo measure rc=$?
