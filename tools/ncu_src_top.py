"""Summarise an `ncu --page source --csv` (SASS view) export: the instructions
with the most stall samples, their dominant stall reasons, and shared-memory
excess wavefronts per instruction.

    python tools/ncu_src_top.py gpurun_out/prof/p6f32v3_src.csv [--top 25]
"""
import argparse
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    recs = []
    tot = 0
    tot_stall = {h: 0 for h in stall_cols}
    excess = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        tot += smp
        st = {h: int(r[ix[h]] or 0) for h in stall_cols}
        for h in stall_cols:
            tot_stall[h] += st[h]
        ex = int(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
        excess += ex
        recs.append((smp, r[ix["Address"]][-5:], r[ix["Source"]].strip(), st, ex))
    print(f"total samples {tot}; shared excess wavefronts {excess}")
    print("stall totals:", ", ".join(f"{h[6:]}={v / max(tot, 1):.2f}" for h, v in
                                      sorted(tot_stall.items(), key=lambda x: -x[1])[:8]))
    for smp, addr, src, st, ex in sorted(recs, key=lambda x: -x[0])[: a.top]:
        top = sorted(st.items(), key=lambda x: -x[1])[:2]
        print(f"{smp:7d} {addr} {src[:60]:60s} " + " ".join(f"{h[6:]}={v}" for h, v in top) + (f" excess={ex}" if ex else ""))
    print("-- top shared-memory excess wavefronts --")
    for smp, addr, src, st, ex in sorted(recs, key=lambda x: -x[4])[:12]:
        if ex:
            print(f"{ex:9d} {addr} {src[:70]}")


if __name__ == "__main__":
    main()
