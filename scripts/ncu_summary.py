"""Summarise ncu captures for profiles/: per-kernel metrics of a `--set full` report and the
per-kernel share of a `gpu__time_duration.sum` launch list.

  python scripts/ncu_summary.py --report gpurun_out/full.ncu-rep --launches gpurun_out/launches.csv \
      --out profiles/round1_ncu_summary.md --traffic-json profiles/ncu_vertex_pass_traffic.json
"""
import argparse
import collections
import csv
import io
import json
import subprocess

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 RED requests"),
    ("lts__d_atomic_input_cycles_active.max.pct_of_peak_sustained_elapsed",
     "hottest L2 slice atomic-input busy %"),
]


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(val) * scale.get(unit, 1)


def report_rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--report")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic-json")
    ap.add_argument("--title", default="ncu summary")
    ap.add_argument("--skip-steps", type=int, default=0,
                    help="launch list: drop everything before the (N+1)-th vertex-pass launch "
                         "(the bench's warm-up steps) and the input generator k_synth")
    a = ap.parse_args()
    lines = [f"# {a.title}", ""]
    traffic = {}
    if a.report:
        hdr, units, rows = report_rows(a.report)
        ix = {h: i for i, h in enumerate(hdr)}
        lines += ["## `ncu --set full` (one launch per kernel; replayed, cold-cache)", ""]
        for r in rows:
            name = r[ix["Kernel Name"]]
            lines.append(f"### {name}")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for key, label in WANT:
                if key in ix and r[ix[key]] != "":
                    lines.append(f"| {label} (`{key}`) | {r[ix[key]]} {units[ix[key]]} |")
            stalls = [(h, float(r[i])) for h, i in ix.items()
                      if h.startswith("smsp__average_warps_issue_stalled_") and
                      h.endswith("_per_issue_active.ratio") and r[i] not in ("", "n/a")]
            stalls.sort(key=lambda t: -t[1])
            top = ", ".join(f"{h.split('stalled_')[1].split('_per_issue')[0]} {v:.2f}"
                            for h, v in stalls[:6])
            lines.append(f"| top stall reasons (cycles per issued instruction) | {top} |")
            lines.append("")
            rd = to_bytes(r[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
            wr = to_bytes(r[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
            traffic.setdefault(name, []).append(rd + wr)
    if a.launches:
        text = open(a.launches).read()
        body = text[text.index('"ID"'):]
        rows = list(csv.reader(io.StringIO(body)))
        hdr = rows[0]
        ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        seen_vp = 0
        for r in rows[1:]:
            if "k_vertex_pass" in r[ik]:
                seen_vp += 1
            if seen_vp <= a.skip_steps or r[ik].startswith(("k_synth", "k_red_peak")):
                continue
            v = float(r[iv].replace(",", ""))
            v = v / 1e3 if r[iu] == "ns" else (v if r[iu] == "us" else v * 1e3)
            name = r[ik].split("(")[0]
            tot[name] += v
            cnt[name] += 1
        allt = sum(tot.values())
        lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum`, serialised, cold-cache)",
                  "", f"Timed steps only (first {a.skip_steps} vertex-pass steps and the input "
                  "generator and the RED-peak diagnostic dropped).", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            lines.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / allt:.1f}% |")
        lines.append("")
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic_json and traffic:
        vp = {k: v for k, v in traffic.items() if "k_vertex_pass" in k}
        if vp:
            k, v = next(iter(vp.items()))
            with open(a.traffic_json, "w") as f:
                json.dump({"kernel": k, "dram_bytes_per_launch": sum(v) / len(v),
                           "source": a.report}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
