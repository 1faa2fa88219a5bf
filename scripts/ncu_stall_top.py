#!/usr/bin/env python3
"""Top instructions by not-issued warp-state samples of the first kernel in an ncu report
(`ncu -i REP --page source --csv --print-source sass`): profiles/r01_sweep_*_stall_top.txt."""
import csv
import io
import subprocess
import sys


def main():
    rep, label = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         check=True, capture_output=True, text=True).stdout
    hdr, recs = None, []
    for r in csv.reader(io.StringIO(raw)):
        if r and r[0] == "Kernel Name":
            if recs:
                break
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) > 5:
            recs.append((r[0][-6:], r[1].strip(), int(r[2] or 0), int(r[3] or 0)))
    tot_all, tot_ni = sum(x[2] for x in recs), sum(x[3] for x in recs)
    print(f"# ncu --set full source page, {label}: warp-state samples {tot_all}, not-issued {tot_ni}")
    print("# top instructions by not-issued samples (address suffix, samples, not-issued, share of not-issued, SASS)")
    for a, src, al, ni in sorted(recs, key=lambda x: -x[3])[:15]:
        print(f"{a}  {al:6d} {ni:6d}  {ni / max(tot_ni, 1):.3f}  {src}")


if __name__ == "__main__":
    main()
