"""Summarise ncu artefacts into profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py gpurun_out/r01_decode_full.ncu-rep ...   -> markdown to stdout
    python tools/summarize_ncu.py --launches gpurun_out/r01_bench_launches.csv
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
    "smsp__mem_tensor_reads_op_utcmma_matrix_c.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    print(f"### {path.split('/')[-1]}\n")
    for r in data:
        name = r[hdr.index("Kernel Name")]
        print(f"- kernel: `{name[:110]}`")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  - {k}: {r[i]} {units[i]}")
        print()


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[h + 1:]:
        name = r[ki].split("(")[0].replace("void elattn_gpu::<unnamed>::", "")
        tot[name] += float(r[vi]) / 1e3
        cnt[name] += 1
    allt = sum(tot.values())
    print(f"### launch list {path.split('/')[-1]} (ncu gpu__time_duration, cold & serialised)\n")
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / allt:.1%} |")
    print()


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        for p in args[1:]:
            launches(p)
    else:
        for p in args:
            rep(p)
