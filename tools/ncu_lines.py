"""Per-source-line stall samples and executed instructions from an ncu report
(`--page source --print-source cuda,sass`), for the kernel at --launch-skip N.

    python tools/ncu_lines.py report.ncu-rep [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    skip = sys.argv[2] if len(sys.argv) > 2 else "0"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    agg, cur, path, hdr = {}, None, "", None
    stall = {}
    for row in r:
        if len(row) > 5 and row[0] == "Line No":
            hdr = row
            sidx = [(i, h[6:]) for i, h in enumerate(row) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if len(row) >= 2 and row[0] == "File Path":
            path = row[1].split("/")[-1]
            continue
        if len(row) < 8 or row[0] == "Line No":
            continue
        if row[0]:
            cur = (path, int(row[0]), row[1].strip()[:90])
            agg.setdefault(cur, [0, 0])
            continue
        if cur is None:
            continue
        try:
            agg[cur][0] += int(row[4] or 0)
            agg[cur][1] += int(row[7] or 0)
            st = stall.setdefault(cur, {})
            for i, h in sidx:
                if i < len(row) and row[i] not in ("", "-"):
                    st[h] = st.get(h, 0) + int(float(row[i]))
        except ValueError:
            pass
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"samples {tot_s}, instructions {tot_i}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        top3 = sorted(stall.get(k, {}).items(), key=lambda kv: -kv[1])[:3]
        why = " ".join(f"{h}={c}" for h, c in top3 if c)
        print(f"{100 * v[0] / tot_s:5.1f}% samp {100 * v[1] / tot_i:5.1f}% inst  {k[0]}:{k[1]}  {k[2][:60]}  [{why}]")


if __name__ == "__main__":
    main()
