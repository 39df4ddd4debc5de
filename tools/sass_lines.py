"""Join an ncu SASS source page (--page source --csv --print-source sass) with
nvdisasm -g line info: per-source-line executed instructions and stall samples.
    python tools/sass_lines.py all.dis <mangled kernel> sass.csv [top]"""
import csv
import re
import sys
from collections import defaultdict


def main(dis, fun, sass_csv, top=40):
    lines, cur, inside = {}, None, False
    for l in open(dis):
        if l.startswith("//--------------------- .text."):
            inside = l.strip().endswith(fun + " --------------------------")
            continue
        if not inside:
            continue
        m = re.match(r'\s*//## File "(.*)", line (\d+)', l)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if m and cur:
            lines[int(m.group(1), 16)] = cur
    rows = list(csv.reader(open(sass_csv)))
    h = rows[1]
    ia, ie, iss = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    agg = defaultdict(lambda: [0, 0])
    tot = [0, 0]
    base = None
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        try:
            a = int(r[ia], 16)
        except ValueError:
            continue
        if base is None:
            base = a  # the page lists absolute addresses, the disassembly offsets
        a -= base
        ex = float(r[ie] or 0)
        st = float(r[iss] or 0)
        key = lines.get(a, ("?", 0))
        agg[key][0] += ex
        agg[key][1] += st
        tot[0] += ex
        tot[1] += st
    src = {}
    for (f, ln) in agg:
        if f not in src:
            try:
                import glob
                path = glob.glob(f"/root/repo/**/{f}", recursive=True)[0]
                src[f] = open(path).read().split("\n")
            except Exception:
                src[f] = []
    for (f, ln), (ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        text = src[f][ln - 1].strip() if 0 < ln <= len(src[f]) else ""
        print(f"{st / tot[1] * 100:5.1f}% stall {ex / tot[0] * 100:5.1f}% inst  {f}:{ln}  {text[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
