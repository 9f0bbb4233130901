#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_relay.py tests/test_reference_suite.py tests/test_wire.py -q --timeout 300 > gpurun_out/relay_c.log 2>&1; echo "rc=$?" >> gpurun_out/relay_c.log
timeout 300 python scripts/compact_time.py > gpurun_out/compact.json 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > gpurun_out/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
