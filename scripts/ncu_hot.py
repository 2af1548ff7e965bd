"""Top stall locations of one kernel in an ncu report (source page, SASS)."""
import csv
import io
import subprocess
import sys


def main(rep, kernel_regex=None, top=30):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel_regex:
        cmd += ["-k", f"regex:{kernel_regex}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # first kernel block only
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    data = []
    for r in rows[hdr_i + 1:]:
        if not r or r[0] == "Kernel Name":
            break
        data.append(r)
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    i_ex = hdr.index("Instructions Executed")
    tot = sum(float(r[i_s] or 0) for r in data)
    print(f"{rep}: {len(data)} SASS lines, {tot:.0f} samples")
    for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:int(top)]:
        s = float(r[i_s] or 0)
        print(f"{r[0][-5:]} {s:7.0f} {100 * s / tot:5.1f}% ex={r[i_ex]:>9s} {r[i_src][:95]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
