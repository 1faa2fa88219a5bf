#!/bin/bash
# Re-run the f4 validation harness and the f1 equilibration curves (one gpurun call).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
( timeout 1200 python scripts/validate_methods.py --L 512 --K 10 --ps 0.3,0.5,0.7,0.85;
  timeout 1200 python scripts/validate_methods.py --L 2048 --K 5 --ps 0.5,0.85 ) > gpurun_out/val_p.jsonl 2> gpurun_out/val_p.err
( timeout 900 python scripts/validate_methods.py --sweep lb --L 512 --K 10;
  timeout 900 python scripts/validate_methods.py --sweep ns --L 512 --K 10 ) > gpurun_out/val_lbns.jsonl 2> gpurun_out/val_lbns.err
( timeout 900 python scripts/equilibration_curves.py;
  timeout 900 python scripts/equilibration_curves.py --L 1024 --spread 10 ) > gpurun_out/equil.jsonl 2> gpurun_out/equil.err
echo done >> gpurun_out/equil.err
