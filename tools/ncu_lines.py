"""Per-CUDA-source-line instruction / stall summary of `ncu --page source --csv --print-source cuda,sass`.
usage: ncu_lines.py file.csv [n]"""
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    ei, wi = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[hi + 1:]:
        if not r or not r[0] or len(r) <= max(ei, wi):
            continue  # SASS rows carry no line number
        try:
            data.append((float(r[ei] or 0), float(r[wi] or 0), r[0], r[1][:100]))
        except ValueError:
            pass
    ti = sum(d[0] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    print(f"total warp-instructions {ti / 1e6:.2f}M  stall samples {ts:.0f}")
    for inst, st, line, src in sorted(data, reverse=True)[:n]:
        print(f"{100 * inst / ti:5.1f}% inst {100 * st / ts:5.1f}% stall  L{line:>5}  {src.strip()}")


if __name__ == "__main__":
    main()
