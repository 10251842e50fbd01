"""Measurement aid: attribute an ncu capture's warp-stall samples to CUDA
source lines.  The ncu SASS page (per-instruction samples) is aligned by
instruction index with `nvdisasm -g` of the same kernel in the in-tree
libmis2.so, whose line-info comments give the (innermost) source line.

usage: python tools/ncu_lines.py REP.ncu-rep [kernel-substring] [top]
"""
import csv, io, os, re, subprocess, sys, tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2204_02934_b200", "libmis2.so")


def sass_lines(kernel_sub):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, capture_output=True)
    out = []
    for f in sorted(os.listdir(d)):
        if not f.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True, text=True).stdout
        sec = None
        cur = None
        for ln in txt.splitlines():
            m = re.match(r"//-+ \.text\.(\S+) -+", ln)
            if m:
                if sec is not None and out:
                    return out
                sec = m.group(1) if kernel_sub in m.group(1) else None
                out = []
                continue
            if sec is None:
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
                out.append(cur)
        if sec is not None and out:
            return out
    return out


def ncu_sass(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    return [(int(r[i_s] or 0), r[i_src]) for r in rows[2:]]


def main():
    rep = sys.argv[1]
    ksub = sys.argv[2] if len(sys.argv) > 2 else "mis2_persistentILi1ELb0"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    lines = sass_lines(ksub)
    samp = ncu_sass(rep)
    print(f"sass instrs: nvdisasm {len(lines)}  ncu {len(samp)}")
    n = min(len(lines), len(samp))
    agg = {}
    tot = 0
    for i in range(n):
        s = samp[i][0]
        tot += s
        key = lines[i] or ("?", 0)
        agg[key] = agg.get(key, 0) + s
    src = {}
    for (f, l) in agg:
        p = os.path.join(ROOT, "paper_2204_02934_b200", "csrc", f)
        if f not in src and os.path.exists(p):
            src[f] = open(p).read().splitlines()
    print(f"total samples {tot}")
    for (f, l), s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        text = src.get(f, [""] * (l + 1))[l - 1].strip() if f in src and 0 < l <= len(src[f]) else ""
        print(f"{100.0 * s / max(tot, 1):5.1f}%  {f}:{l:<5d} {text[:90]}")


if __name__ == "__main__":
    main()
