#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_relay.py -q --timeout 300 > gpurun_out/relay_d.log 2>&1; echo "rc=$?" >> gpurun_out/relay_d.log
