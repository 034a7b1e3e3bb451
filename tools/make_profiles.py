"""Copy the judged evidence from gpurun_out/ (scratch) into profiles/ (tracked), with summaries.

usage: python tools/make_profiles.py r01
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def jline(path):
    if not os.path.exists(path):
        return None
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            return json.loads(line)
    return None


def launches_summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out, tot = [], {}
    for r in rows[1:]:
        name = r[iN].split("(")[0].replace("void ", "")
        ns = float(r[iV])
        out.append((name, ns))
        tot[name] = tot.get(name, 0.0) + ns
    return out, tot


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(P, exist_ok=True)
    md = [f"# Profiles and bench evidence, round {tag}\n",
          "All numbers below come from `tools/run_evidence.sh` on one B200 (gpurun). ncu runs used "
          "`--clock-control none`; a number measured under ncu is never a bench value.\n"]
    for name in ("bench_final", "bench_ref", "bench_c3_q64", "bench_c3v", "bench_c3v_dense",
                 "bench_c4v_n1", "bench_c5", "bench_c2", "bench_c2_grad"):
        d = jline(os.path.join(G, f"{name}.json"))
        if d is None:
            continue
        json.dump(d, open(os.path.join(P, f"{tag}_{name}.json"), "w"), indent=1)
        md.append(f"## {name}: {d.get('config', {}).get('workload', '')}\n")
        md.append(f"* value **{d['value']:.6g} {d['unit']}**, ms/step {d['ms_per_step']:.4g}")
        if "roofline" in d:
            r = d["roofline"]
            md.append(f"* roofline: {r['achieved']:.1f} / {r['peak']} {r['unit']} = **{r['frac']:.3f}** "
                      f"({r.get('peak_source', '')}); traffic/launch {r.get('traffic')}; kernel share of "
                      f"step {r.get('kernel_share_of_step', 0):.3f}")
        if d.get("e2e"):
            md.append(f"* e2e: {d['e2e']['value']:.6g} {d['e2e']['unit']} (H2D {d['e2e']['h2d_bytes_per_step']} B, "
                      f"D2H {d['e2e']['d2h_bytes_per_step']} B per step)")
        if d.get("clocks"):
            md.append(f"* clocks: {d['clocks']}")
        if d.get("cpu_baseline"):
            c = d["cpu_baseline"]
            md.append(f"* cpu_baseline ({c['kind']}, {c['cores']} cores): {c['value']:.4g} {c['unit']} -- {c['sample']}")
        md.append("")
    lp = os.path.join(G, "launches.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(P, f"{tag}_launches.csv"))
        seq, tot = launches_summary(lp)
        md.append("## Launch list (ncu gpu__time_duration.sum, `bench.py --steps 2 --warmup 1`)\n")
        md.append("Cold-cache, serialised times; compare shares, not absolutes.\n")
        md.append("| kernel | total ms | share of timed-loop kernels |\n|---|---|---|")
        loop = {k: v for k, v in tot.items() if "hiper::" in k}
        s = sum(loop.values()) or 1.0
        for k, v in sorted(loop.items(), key=lambda x: -x[1]):
            md.append(f"| {k} | {v / 1e6:.3f} | {v / s:.4f} |")
        md.append("")
    tp = os.path.join(G, "traffic.csv")
    if os.path.exists(tp):
        shutil.copy(tp, os.path.join(P, f"{tag}_traffic.csv"))
        vals = {}
        for r in csv.reader(open(tp)):
            if len(r) > 14 and r[12].startswith(("dram", "gpu__", "lts")):
                vals[r[12]] = float(r[14])
        bench = jline(os.path.join(G, "bench_final.json")) or {}
        cfg = bench.get("config", {})
        dram = vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0)
        ent = {"dram_bytes_per_launch": dram, "dram_read": vals.get("dram__bytes_read.sum"),
               "dram_write": vals.get("dram__bytes_write.sum"), "lts_bytes": vals.get("lts__t_bytes.sum"),
               "duration_ns_under_ncu": vals.get("gpu__time_duration.sum"),
               "chunks_per_gpu": cfg.get("corpus_per_gpu"), "queries": cfg.get("query_batch"),
               "source": f"profiles/{tag}_traffic.csv: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                         "--replay-mode application on `bench.py --steps 2 --warmup 1` (one launch)"}
        json.dump({"maxsim_sm100_kernel": ent}, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
        alg = (cfg.get("corpus_per_gpu") or 0) * cfg.get("chunk_len", 0) * cfg.get("dim", 0) * 2
        md.append("## DRAM traffic of one fused-kernel launch of the bench workload\n")
        md.append(f"* dram read+write {dram / 1e9:.1f} GB per launch; algorithmic (corpus once) "
                  f"{alg / 1e9:.1f} GB -> {dram / max(alg, 1):.2f}x")
        md.append(f"* L2 (lts) bytes {vals.get('lts__t_bytes.sum', 0) / 1e12:.2f} TB\n")
    sp = os.path.join(G, "pipe_stats.log")
    if os.path.exists(sp):
        lines = sorted(set(l.strip() for l in open(sp) if l.startswith("[hiper pipe]")))
        open(os.path.join(P, f"{tag}_pipe_stats.txt"), "w").write("\n".join(lines) + "\n")
        md.append("## Pipeline statistics (HIPER_PIPE_STATS=1, 300k-chunk runs of config3 / config3v / config5)\n")
        md.append("MMA-thread waits are issue-side (the tensor pipe may still be busy); drain = cycles an "
                  "epilogue warp holds an accumulator after it is full.\n\n```\n" + "\n".join(lines) + "\n```\n")
    for rep, label in (("prof_final", "fused MaxSim kernel, config-3 shape at C=100k"),
                       ("prof_packed", "fused MaxSim kernel on the packed layout (N4), config3v at C=200k"),
                       ("prof_pooled", "pooled kernel, config-5 full size (3.6M x 768, Q=4096)")):
        rp = os.path.join(G, f"{rep}.ncu-rep")
        if os.path.exists(rp):
            shutil.copy(rp, os.path.join(P, f"{tag}_{rep}.ncu-rep"))
            txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), rp, "20"],
                                 capture_output=True, text=True).stdout
            open(os.path.join(P, f"{tag}_{rep}_summary.txt"), "w").write(txt)
            md.append(f"## ncu --set full: {label}\n\n```\n{txt}\n```\n")
    for f in ("pytest_gpu.log", "smoke.log"):
        fp = os.path.join(G, f)
        if os.path.exists(fp):
            shutil.copy(fp, os.path.join(P, f"{tag}_{f}"))
    open(os.path.join(P, f"{tag}_SUMMARY.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
