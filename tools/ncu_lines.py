"""Per-source-line summary of an ncu report (--import-source on capture):
warp-stall samples and executed warp instructions by CUDA line, plus the
SASS of the hottest lines.

    python tools/ncu_lines.py report.ncu-rep [--top 40] [--sass LINE ...]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    per_line = defaultdict(lambda: [0, 0, ""])
    sass = defaultdict(list)
    cur_file, cur_line, hdr = "", None, None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0] != "-" and r[0] != "":
            cur_line = (cur_file, int(r[0]))
            per_line[cur_line][2] = r[1]
        elif cur_line is not None:
            # SASS row: Address, Source, stall all, stall not issued, samples, inst executed
            try:
                st, ins = int(r[4]), int(r[7])
            except ValueError:
                continue
            per_line[cur_line][0] += st
            per_line[cur_line][1] += ins
            sass[cur_line].append((r[3], st, ins))
    return per_line, sass


def main():
    rep = sys.argv[1]
    top = 40
    show = []
    a = sys.argv[2:]
    if "--top" in a:
        top = int(a[a.index("--top") + 1])
    if "--sass" in a:
        show = [int(v) for v in a[a.index("--sass") + 1:]]
    per_line, sass = load(rep)
    tot_s = sum(v[0] for v in per_line.values()) or 1
    tot_i = sum(v[1] for v in per_line.values()) or 1
    print(f"total stall samples {tot_s}, warp instructions {tot_i}")
    for key, (st, ins, src) in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*st/tot_s:5.1f}% stall {100*ins/tot_i:5.1f}% inst  {key[0]}:{key[1]:<5d} "
              f"{src.strip()[:90]}")
    for ln in show:
        for key in per_line:
            if key[1] == ln and key[0].endswith(".cu"):
                print(f"--- {key[0]}:{ln}")
                for s, st, ins in sass[key]:
                    print(f"   {st:7d} {ins:11d}  {s}")


if __name__ == "__main__":
    main()


def dump_sass(rep, path):
    """Every SASS instruction of the report with its CUDA line, stall samples
    and executed count, in address order."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    with open(path, "w") as f:
        for r in rows:
            if len(r) > 8 and r[0].startswith("0x"):
                f.write(f"{r[0][-5:]} {int(r[2]):7d} {int(r[5]):11d}  {r[1]}\n")
