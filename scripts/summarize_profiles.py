"""Summarise one gpu_round.sh session into profiles/ (tracked).

    python scripts/summarize_profiles.py TAG ROUND [OUTDIR]

reads gpurun_out/TAG_{launches.csv,csr.ncu-rep,cg.ncu-rep,bench.json,
bench_ref.json,pytest_gpu.log} and writes profiles/rROUND_launches_summary.txt,
rROUND_csr_stream_ncu_full.txt, rROUND_cg_kernels_ncu.txt,
rROUND_bench_N1.json, rROUND_bench_reference_N1.json and ncu_summary.json
(the roofline `traffic` source read by bench.py)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, rnd = sys.argv[1], int(sys.argv[2])  # noqa: E501
G = os.path.join(ROOT, "gpurun_out")
args = [a for a in sys.argv[1:] if not a.startswith("--")]
P = args[2] if len(args) > 2 else os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)
CSR_BYTES = 710858660  # cfg2: 12 nnz + 4 (n + 1) + 16 n

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic"]


def launches():
    rows = list(csv.reader(open(os.path.join(G, f"{tag}_launches.csv"))))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                 "msecond": 1e3}
        us = v * scale[d["Metric Unit"]]
        a = agg.setdefault(d["Kernel Name"], [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py "
           f"--steps 20 --warmup 3 --no-cpu --no-formats",
           "# cold-cache, serialised launches: compare SHARES, not absolutes. First 400 launches: "
           "device stencil gen, bench SpMV steps (cfg2), e2e steps, then the CG cfg4 kernels.",
           "launches     total_us     avg_us  share  kernel"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{n:8d} {us:12.1f} {us / n:10.1f} {100 * us / tot:5.1f}%  {k}")
    open(os.path.join(P, f"r{rnd}_launches_summary.txt"), "w").write("\n".join(out) + "\n")


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    return [(dict(zip(h, r)), dict(zip(h, units))) for r in rows[2:] if len(r) == len(h)]


def fmt(d, u, m):
    return f"{m} = {d.get(m, '?')} {u.get(m, '')}".rstrip()


def to_bytes(d, u, m):
    v = float(d[m].replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u[m], 1)


def csr_full():
    rep = os.path.join(G, f"{tag}_csr.ncu-rep")
    (d, u), = raw(rep)[:1]
    dram = to_bytes(d, u, "dram__bytes_read.sum") + to_bytes(d, u, "dram__bytes_write.sum")
    dur = float(d["gpu__time_duration.sum"].replace(",", ""))
    dur_us = dur / 1e3 if u["gpu__time_duration.sum"] == "nsecond" else dur
    lines = ["# ncu --set full --clock-control none --import-source on -k regex:csr_stream -s 5 "
             "-c 1 python bench.py --steps 8 --warmup 3 --no-cg --no-cpu --no-formats",
             f"# kernel: {d['Kernel Name']}",
             f"# workload: cfg2 CSR SpMV (27-pt 128^3, 55,742,968 nnz); algorithmic bytes/launch "
             f"{CSR_BYTES:,}"]
    lines += [fmt(d, u, m) for m in METRICS]
    lines.append(f"dram_bytes_total = {int(dram)} B  (traffic / algorithmic = "
                 f"{dram / CSR_BYTES:.3f}; x is L2-resident)")
    open(os.path.join(P, f"r{rnd}_csr_stream_ncu_full.txt"), "w").write("\n".join(lines) + "\n")
    json.dump({"round": rnd, "source": f"profiles/r{rnd}_csr_stream_ncu_full.txt",
               "kernels": {"csr_stream_kernel": {
                   "config": "cfg2", "dram_bytes_per_launch": int(dram),
                   "algorithmic_bytes_per_launch": CSR_BYTES, "ncu_duration_us": dur_us}}},
              open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)


def cg_full():
    rep = os.path.join(G, f"{tag}_cg.ncu-rep")
    if not os.path.exists(rep):
        return
    lines = ["# ncu --set full --clock-control none -k regex:'csr_stream|vec_kernel' "
             "python scripts/prof_k1.py: plain cfg4 CSR SpMV, then 2 CG iterations (cfg4, 7-pt "
             "256^3): EpiInit, K1, K2, K3"]
    for d, u in raw(rep):
        lines.append(f"\n[{d['Kernel Name'][:150]}]")
        lines += ["  " + fmt(d, u, m) for m in METRICS]
    open(os.path.join(P, f"r{rnd}_cg_kernels_ncu.txt"), "w").write("\n".join(lines) + "\n")


def cfg3_full():
    """cfg3 power-law captures (TAG_pl_{csr,coo,f32}.ncu-rep, one launch each,
    scripts/prof_pl.py) -> rROUND_cfg3_ncu.txt and ncu_summary.json entries."""
    n, nnz = 1 << 24, 268_195_029
    alg = {"csr": 12 * nnz + 4 * (n + 1) + 16 * n, "coo": 16 * nnz + 16 * n,
           "f32": 8 * nnz + 4 * (n + 1) + 8 * n}
    lines = ["# ncu --set full --clock-control none -k regex:'csr_stream|coo_stream' -c 1 "
             "python scripts/prof_pl.py {csr|coo|f32}: cfg3 power-law (2^24 rows, 268,195,029 "
             "nnz, max row 10,000), one launch each"]
    summ = json.load(open(os.path.join(P, "ncu_summary.json")))
    found = False
    for w in ("csr", "coo", "f32"):
        rep = os.path.join(G, f"{tag}_pl_{w}.ncu-rep")
        if not os.path.exists(rep):
            continue
        found = True
        (d, u), = raw(rep)[:1]
        dram = to_bytes(d, u, "dram__bytes_read.sum") + to_bytes(d, u, "dram__bytes_write.sum")
        dur = float(d["gpu__time_duration.sum"].replace(",", ""))
        dur_us = dur / 1e3 if u["gpu__time_duration.sum"] == "nsecond" else dur
        lines.append(f"\n[cfg3 {w}: {d['Kernel Name'][:120]}]")
        lines += ["  " + fmt(d, u, m) for m in METRICS]
        lines.append(f"  dram_bytes_total = {int(dram)} B  (traffic / algorithmic = "
                     f"{dram / alg[w]:.3f})")
        summ["kernels"][f"cfg3_{w}"] = {
            "config": f"cfg3 {w}", "kernel": d["Kernel Name"][:120],
            "dram_bytes_per_launch": int(dram), "algorithmic_bytes_per_launch": alg[w],
            "ncu_duration_us": dur_us,
            "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
            "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
            "l1_lsu_wavefronts_pct": float(
                d["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]),
            "source": f"profiles/r{rnd}_cfg3_ncu.txt"}
    if found:
        open(os.path.join(P, f"r{rnd}_cfg3_ncu.txt"), "w").write("\n".join(lines) + "\n")
        json.dump(summ, open(os.path.join(P, "ncu_summary.json"), "w"), indent=1)


def bench():
    for src, dst in ((f"{tag}_bench.json", f"r{rnd}_bench_N1.json"),
                     (f"{tag}_bench_ref.json", f"r{rnd}_bench_reference_N1.json")):
        lines = [ln for ln in open(os.path.join(G, src)).read().splitlines()
                 if ln.startswith("{")]
        if lines:
            json.dump(json.loads(lines[-1]), open(os.path.join(P, dst), "w"), indent=1)


if "--cfg3-only" in sys.argv:
    cfg3_full()
    print("ok")
    sys.exit(0)
launches()
if "--launches-only" not in sys.argv:
    csr_full()
    cg_full()
    bench()
print("ok")
