"""Summarise `ncu --page source --csv` (SASS) output.
usage: ncu_sass_top.py file.csv [section_index] [mode: top|blocks] [n]"""
import csv
import sys


def sections(path):
    secs, cur = [], None
    for r in csv.reader(open(path)):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": [], "h": None}
            secs.append(cur)
        elif cur is not None:
            if cur["h"] is None and "Address" in r:
                cur["h"] = r
            elif cur["h"] is not None:
                cur["rows"].append(r)
    return secs


def main():
    secs = sections(sys.argv[1])
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    mode = sys.argv[3] if len(sys.argv) > 3 else "top"
    n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    s = secs[k]
    h = s["h"]
    ai, si = h.index("Address"), h.index("Source")
    wi, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = []
    for r in s["rows"]:
        try:
            data.append((r[ai][-5:], int(r[ei] or 0), int(r[wi] or 0), r[si].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[2] for d in data) or 1
    ti = sum(d[1] for d in data) or 1
    print(f"{s['name'][:90]}\nsamples {tot} warp-instructions {ti} sass lines {len(data)}")
    if mode == "top":
        for d in sorted(data, key=lambda x: -x[2])[:n]:
            print(f"{d[2] / tot * 100:5.1f}%  {d[1]:>10}  {d[0]}  {d[3][:90]}")
    else:
        for i in range(0, len(data), n):
            ch = data[i:i + n]
            ops = " ".join(d[3].split()[0] for d in ch if d[1] > ti * 0.002)[:110]
            print(f"{ch[0][0]} inst={sum(d[1] for d in ch) / ti * 100:5.1f}% samp={sum(d[2] for d in ch) / tot * 100:5.1f}%  {ops}")


if __name__ == "__main__":
    main()
