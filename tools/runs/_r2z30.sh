timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2z30_pytest.log 2>&1; tail -3 gpurun_out/r2z30_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
