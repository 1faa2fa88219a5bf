#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python scripts/f1_equilibrium.py --corr-len 2 > gpurun_out/f1_equilibrium_cl2.jsonl 2> gpurun_out/f1_equilibrium_cl2.err; echo "rc=$?" >> gpurun_out/f1_equilibrium_cl2.err
timeout 1500 python scripts/f1_equilibrium.py --corr-len 1 --sizes 2048,8192 --ps 0.3 > gpurun_out/f1_equilibrium_cl1.jsonl 2> gpurun_out/f1_equilibrium_cl1.err; echo "rc=$?" >> gpurun_out/f1_equilibrium_cl1.err
