"""Top SASS instructions by warp-stall samples from
`ncu -i REP --page source --csv --print-source sass` output (first kernel
or the one matching argv[2])."""
import csv
import io
import sys


def main(path, match="", top=30):
    text = open(path).read()
    blocks = text.split('"Kernel Name",')
    for blk in blocks[1:]:
        name = blk.split("\n", 1)[0]
        if match and match not in name:
            continue
        rows = list(csv.reader(io.StringIO(blk.split("\n", 1)[1])))
        h = rows[0]
        si = h.index("Warp Stall Sampling (All Samples)")
        ie = h.index("Instructions Executed")
        data = [(int(r[si] or 0), r[0], r[1], r[ie]) for r in rows[1:] if len(r) > si]
        tot = sum(d[0] for d in data)
        print(name[:100], "total samples", tot)
        for i, (s, addr, src, ex) in enumerate(data):
            pass
        for s, addr, src, ex in sorted(data, reverse=True)[:top]:
            print(f"{s:6d} {100 * s / max(1, tot):5.1f}%  exec={ex:>8}  {addr[-5:]}  {src.strip()[:90]}")
        break


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "", int(sys.argv[3]) if len(sys.argv) > 3 else 30)
