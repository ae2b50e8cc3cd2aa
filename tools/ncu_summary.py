"""Summarise ncu launch lists (profiles/*_launches_*.csv, captured with
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv
        --log-file <csv> python bench.py --config <cfg> ...)
into profiles/ncu_r2.json: per config, the projection and attention kernels' average cold-cache launch duration
and DRAM bytes per launch, stamped with the sha256 of the library binary the capture ran and the digest of the sources it was
built from (bench.py uses an entry when either matches: nvcc builds are not bit-reproducible).

    python tools/ncu_summary.py <config>=<csv> ... [--lib paper_2511_06077_b200/libstca.so]
"""
import argparse
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kernel_rows(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    head = rows[h]
    ik, im, iv = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value")
    iu = head.index("Metric Unit")
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,  # -> ms
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    iid = head.index("ID")
    per = {}
    for r in rows[h + 1:]:
        if len(r) <= iv:
            continue
        d = per.setdefault(r[iid], {"name": r[ik]})
        try:
            d[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        except ValueError:
            pass
    return list(per.values())


def summarise(path):
    out = {}
    for key, pat in (("project", "k_tc_project"), ("attention", "attention")):
        ks = [k for k in kernel_rows(path) if pat in k["name"]]
        if not ks:
            continue
        n = len(ks)
        dur_ms = sum(k.get("gpu__time_duration.sum", 0.0) for k in ks) / n
        rd = sum(k.get("dram__bytes_read.sum", 0.0) for k in ks) / n
        wr = sum(k.get("dram__bytes_write.sum", 0.0) for k in ks) / n
        out[key] = {"kernel": ks[0]["name"].split("(")[0], "launches": n, "ms_per_launch": dur_ms,
                    "dram_bytes_read_per_launch": rd, "dram_bytes_write_per_launch": wr}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("pairs", nargs="+")
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_2511_06077_b200", "libstca.so"))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_r2.json"))
    ap.add_argument("--lib-sha", default=None, help="the binary's sha256 if the capture ran another build of the "
                                                    "same sources")
    a = ap.parse_args()
    sha = hashlib.sha256(open(a.lib, "rb").read()).hexdigest()
    sys.path.insert(0, ROOT)
    from paper_2511_06077_b200 import build as _b  # noqa: E402
    src = _b.source_digest()
    res = json.load(open(a.out)) if os.path.exists(a.out) else {}
    for p in a.pairs:
        cfg, path = p.split("=", 1)
        res[cfg] = {"lib_sha256": sha if a.lib_sha is None else a.lib_sha, "src_sha256": src,
                    "source": os.path.relpath(path, ROOT), **summarise(path)}
    json.dump(res, open(a.out, "w"), indent=1)
    json.dump(res, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
