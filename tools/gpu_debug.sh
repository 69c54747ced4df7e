#!/bin/bash
mkdir -p gpurun_out
python tools/debug_colour.py > gpurun_out/debug.log 2>&1
SPHP_MAX_GRID=4 python tools/debug_colour.py >> gpurun_out/debug.log 2>&1
