#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 300 python tools/dbg_resident.py > $O/r2h_dbg.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/r2h_all.log 2>&1; echo rc=$? >> $O/r2h_all.log
