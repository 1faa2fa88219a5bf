#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rc in 2 4 8; do MPR_DC_RC=$rc timeout 600 python scripts/micro/order_timing.py 2>&1 | grep "dc tiled=1" | sed "s/^/rc=$rc /"; done > gpurun_out/order_timing2.log
