"""Markdown summary of an ncu report (`ncu -i X.ncu-rep --page raw --csv`), for profiles/.

    python tools/ncu_summary.py gpurun_out/adv_r01c.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units = r[0], r[1]
    return [(dict(zip(head, x)), dict(zip(head, units))) for x in r[2:]]


def main():
    for path in sys.argv[1:]:
        for d, u in rows(path):
            print(f"### {path}: `{d.get('Kernel Name', '?')[:110]}`\n")
            print("| metric | value |\n|---|---|")
            for k, name in KEYS:
                if k in d:
                    print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
            stalls = []
            for k, v in d.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len(
                            "_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            print("| top stalls (warps per issue) | " + ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]) + " |\n")


if __name__ == "__main__":
    main()
