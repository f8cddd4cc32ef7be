"""Per-kernel SASS evidence of the Blackwell-native instruction mix.

`cuobjdump -sass libemm.so`, split by function, counting the mnemonics that
prove the tcgen05 / TMA / TMEM path (B200_PROFILING.md): UTCHMMA (tcgen05.mma,
.2CTA = cta_group::2), UTMALDG / UTMASTG (TMA tensor loads / stores), UBLKCP
(1-D bulk copies), LDTM / STTM (tcgen05.ld / st), UTCBAR (tcgen05.commit),
SYNCS (mbarrier), plus the legacy HMMA (mma.sync) and LDGSTS (cp.async) so the
kernels that deliberately stay on them (decode attention) are visible too.

    python tools/sass_counts.py [lib.so] > profiles/r02/sass_counts.txt
"""
import collections
import os
import re
import subprocess
import sys

MNEMONICS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "UTMACCTL", "UBLKCP",
             "LDTM", "STTM", "SYNCS", "HMMA", "LDGSTS", "MUFU.EX2", "FFMA2", "FADD2", "FMUL2"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True,
                             check=True).stdout.splitlines()
        return dict(zip(names, out))
    except Exception:
        return {n: n for n in names}


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
        os.path.dirname(__file__), "..", "paper_2507_10069_b200", "libemm.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                          check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        op = m.group(1)
        counts[cur]["total"] += 1
        for key in MNEMONICS:
            if op == key or op.startswith(key + "."):
                counts[cur][key if key != "UTCHMMA" or ".2CTA" not in op else "UTCHMMA.2CTA"] += 1
    names = demangle(list(counts))
    print(f"# cuobjdump -sass {os.path.basename(lib)} (sm_100a): instruction counts per kernel")
    cols = ["total"] + [k for k in MNEMONICS + ["UTCHMMA.2CTA"]
                        if any(c[k] for c in counts.values())]
    print("kernel\t" + "\t".join(cols))
    for name, c in sorted(counts.items(), key=lambda kv: names[kv[0]]):
        short = re.sub(r"\(.*", "", names[name]).replace("emm::", "")
        tmpl = re.search(r"<[^()]*>", names[name])
        if tmpl and tmpl.group(0) not in short:
            short += tmpl.group(0)
        print(short + "\t" + "\t".join(str(c[k]) for k in cols))


if __name__ == "__main__":
    main()
