#!/bin/bash
O=gpurun_out; mkdir -p $O
timeout 600 python tools/dbg_resident.py > $O/r2i_dbg.log 2>&1
