"""Summarise tools/evidence.sh output into profiles/<tag>_counters.txt and
profiles/<tag>_sass/<kernel>.txt (SASS with per-instruction executed counts
and stall samples from the ncu source page; HOT marks the hot loops).

    python tools/evidence_summary.py r02 [--n 1000000 --nc 934848 --P 13674493 --npix 2073600]

Per kernel of the second training iteration at config B:
  * duration, warp instructions and the ISSUE roofline: the time the kernel's
    warp instructions need at one issue per cycle on each of the 4 x 148
    schedulers at the measured SM clock, and its fraction of the duration;
  * the byte-model HBM fraction (SURVEY 8(d) algorithmic bytes / duration /
    MEASURED_PEAKS hbm_gbs) beside the measured DRAM traffic;
  * atomics (L1 / L2 RED requests and sectors, L2 atomic-unit utilisation),
    branch efficiency (uniform / all branch targets, SIMT thread efficiency),
    MUFU (XU pipe) utilisation, FMA / ALU pipe utilisation, shared-memory
    bank conflicts.
"""
import argparse
import csv
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

OURS = ("project_cull_compact", "tile_count", "scan_local", "scan_finish", "st_scatter", "st_sort_emit",
        "raster_fwd", "loss_kernel", "raster_bwd", "chain_kernel", "adam_kernel")


def model_bytes(name, n, nc, P, npix):
    """SURVEY 8(d) algorithmic bytes per launch (binning split by stage)."""
    if "project_cull_compact" in name:
        return 56 * n + 48 * nc
    if "tile_count" in name:
        return 48 * nc + 36 * nc
    if "scan_" in name:
        return None
    if "st_scatter" in name:
        return 48 * nc
    if "st_sort_emit" in name:
        return 4 * P
    if "raster_fwd" in name:
        return 40 * P + 20 * npix
    if "loss_kernel" in name:
        return 36 * npix
    if "raster_bwd" in name:
        return 96 * P + 20 * npix
    if "chain_kernel" in name:
        return 188 * nc
    if "adam_kernel" in name:
        return 400 * nc
    return None


def metrics(tag):
    rows = [r for r in csv.reader(open(os.path.join(OUT, f"{tag}_metrics.csv"))) if len(r) > 10]
    h = rows[0]
    per = OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (int(d["ID"]), d["Kernel Name"])
        per.setdefault(key, {})[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    return per


def val(m, k, scale_unit=True):
    if k not in m:
        return None
    v, u = m[k]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    if scale_unit:
        x *= {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
              "second": 1.0, "byte": 1, "Kbyte": 1e3,
              "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
    return x


def counters(tag, a, peak):
    per = metrics(tag)
    # the second iteration: the last occurrence of each of our kernels
    last = OrderedDict()
    for (i, name), m in per.items():
        short = name.split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        if any(o in short for o in OURS):
            last[short] = m
    lines = [f"# {tag}: ncu --metrics pass (tools/evidence.sh), second training iteration at config B "
             f"(N={a.n}, N_c={a.nc}, P={a.P}, Npix={a.npix}); peak HBM {peak} GB/s (MEASURED_PEAKS.json).",
             "# issue roofline = warp instructions / (4 schedulers x 148 SMs x measured SM clock); "
             "frac = roofline time / duration.",
             "# byte model = SURVEY 8(d) algorithmic bytes; dram = measured DRAM read + write.", ""]
    tot_t = tot_issue = 0.0
    for k, m in last.items():
        t = val(m, "gpu__time_duration.sum")
        inst = val(m, "smsp__inst_executed.sum", False)
        cyc = val(m, "sm__cycles_elapsed.avg", False)
        clk = cyc / t if t and cyc else 1.965e9
        t_issue = inst / (4 * 148 * clk) if inst else None
        mb = model_bytes(k, a.n, a.nc, a.P, a.npix)
        dram = (val(m, "dram__bytes_read.sum") or 0) + (val(m, "dram__bytes_write.sum") or 0)
        lines.append(f"== {k}")
        lines.append(f"   duration {t * 1e6:9.1f} us   SM clock {clk / 1e9:.3f} GHz   warp instructions {inst:,.0f}")
        if t_issue:
            lines.append(f"   issue roofline {t_issue * 1e6:9.1f} us  -> {t_issue / t:.2f} of the issue bound "
                         f"(issue active {val(m, 'smsp__issue_active.avg.pct_of_peak_sustained_active', False):.1f}%, "
                         f"warps/SM {val(m, 'sm__warps_active.avg.per_cycle_active', False):.1f})")
            tot_t += t
            tot_issue += t_issue
        if mb:
            lines.append(f"   byte model {mb / 1e6:9.1f} MB -> {mb / t / 1e9:7.1f} GB/s = {mb / t / 1e9 / peak:.3f} "
                         f"of HBM peak;  dram {dram / 1e6:.1f} MB ({dram / mb:.3f} of the model), "
                         f"L2 hit {val(m, 'lts__t_sector_hit_rate.pct', False):.1f}%")
        else:
            lines.append(f"   dram {dram / 1e6:.1f} MB, L2 hit {val(m, 'lts__t_sector_hit_rate.pct', False):.1f}%")
        red_rq = val(m, "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", False) or 0
        red_sec = val(m, "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum", False) or 0
        l2_red = val(m, "lts__t_requests_srcunit_tex_op_red.sum", False) or 0
        l2_red_s = val(m, "lts__t_sectors_srcunit_tex_op_red.sum", False) or 0
        atom = val(m, "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", False) or 0
        if red_rq or atom:
            lines.append(f"   atomics: RED requests L1 {red_rq:,.0f} ({red_sec:,.0f} sectors), L2 {l2_red:,.0f} "
                         f"({l2_red_s:,.0f} sectors), ATOM requests {atom:,.0f}; L2 atomic unit active "
                         f"{val(m, 'lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed', False):.1f}%"
                         f" of elapsed")
        bt = val(m, "smsp__sass_branch_targets.sum", False) or 0
        bd = val(m, "smsp__sass_branch_targets_threads_divergent.sum", False) or 0
        bu = val(m, "smsp__sass_branch_targets_threads_uniform.sum", False) or 0
        simt = val(m, "smsp__thread_inst_executed_per_inst_executed.ratio", False) or 0
        if bt:
            lines.append(f"   branches: {bt:,.0f} targets, {bd:,.0f} divergent -> branch efficiency "
                         f"{bu / bt * 100:.1f}% uniform; SIMT efficiency {simt:.2f}/32 threads per instruction")
        lines.append(f"   pipes: MUFU (XU) {val(m, 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', False):.1f}%"
                     f" of peak ({val(m, 'smsp__inst_executed_pipe_xu.sum', False):,.0f} warp instr), FMA "
                     f"{val(m, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active', False):.1f}%, ALU "
                     f"{val(m, 'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', False):.1f}%; "
                     f"shared bank conflicts "
                     f"{val(m, 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', False):,.0f} of "
                     f"{val(m, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', False):,.0f} wavefronts")
        lines.append("")
    lines.append(f"Iteration kernels: {tot_t * 1e6:.1f} us measured, {tot_issue * 1e6:.1f} us issue-bound floor "
                 f"({tot_issue / tot_t:.2f})")
    return "\n".join(lines) + "\n"


CALLS = {"sb_project_cull_compact": ("project_cull_compact",), "sb_bin_prepare": ("tile_count", "scan_local",
                                                                                    "scan_finish"),
         "sb_bin_finish": ("st_scatter", "st_sort_emit"), "sb_raster_fwd": ("raster_fwd",),
         "sb_loss_fwd_bwd": ("loss_kernel",), "sb_raster_bwd": ("raster_bwd",),
         "sb_chain_projection_bwd": ("chain_kernel",), "sb_adam_sparse": ("adam_kernel",)}


def traffic_json(tag):
    """profiles/traffic.json: per C-ABI call, the capture's DRAM bytes and warp
    instructions (bench.py reports them beside its live timings)."""
    per = metrics(tag)
    last = OrderedDict()
    for (i, name), m in per.items():
        short = name.split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        last[short] = m
    out = {"_source": f"profiles/{tag}_counters.txt: ncu --metrics pass (tools/evidence.sh {tag}), config B, "
                      "second training iteration; dram = dram__bytes_read.sum + dram__bytes_write.sum, "
                      "warp_instructions = smsp__inst_executed.sum, summed over the call's kernels"}
    for call, ks in CALLS.items():
        d = w = 0.0
        for short, m in last.items():
            if any(k in short for k in ks):
                d += (val(m, "dram__bytes_read.sum") or 0) + (val(m, "dram__bytes_write.sum") or 0)
                w += val(m, "smsp__inst_executed.sum", False) or 0
        out[call] = {"dram_bytes": d, "warp_instructions": w}
    with open(os.path.join(PROF, "traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def sass_pages(tag):
    os.makedirs(os.path.join(PROF, f"{tag}_sass"), exist_ok=True)
    for f in sorted(os.listdir(OUT)):
        if not (f.startswith(f"{tag}_full_") and f.endswith(".ncu-rep")):
            continue
        k = f[len(f"{tag}_full_"):-len(".ncu-rep")]
        txt = subprocess.run(["ncu", "-i", os.path.join(OUT, f), "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
        if not hi:
            continue
        h = rows[hi[0]]
        data = [dict(zip(h, r)) for r in rows[hi[0] + 1:(hi[1] if len(hi) > 1 else None)] if len(r) == len(h)]

        def I(d, key):
            try:
                return int(d[key])
            except (KeyError, ValueError):
                return 0
        mx = max(I(d, "Instructions Executed") for d in data) or 1
        tot = sum(I(d, "Instructions Executed") for d in data)
        smp = sum(I(d, "Warp Stall Sampling (All Samples)") for d in data) or 1
        out = [f"# {k}: SASS (sm_100a) from ncu --page source --print-source sass, config B second iteration",
               f"# columns: HOT marker (executed >= 25% of the hottest instruction), warp instructions executed,",
               f"#          stall samples (% of {smp}), address, instruction.  Total warp instructions {tot:,}.",
               ""]
        for d in data:
            n = I(d, "Instructions Executed")
            s = I(d, "Warp Stall Sampling (All Samples)")
            mark = "HOT" if n >= 0.25 * mx else "   "
            out.append(f"{mark} {n:>11,} {100.0 * s / smp:5.1f}%  {d['Address'][-6:]}  {d['Source'].strip()}")
        with open(os.path.join(PROF, f"{tag}_sass", f"{k}.txt"), "w") as fh:
            fh.write("\n".join(out) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--nc", type=int, default=934_848)
    ap.add_argument("--P", type=int, default=13_674_493)
    ap.add_argument("--npix", type=int, default=1920 * 1080)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    with open(os.path.join(PROF, f"{a.tag}_counters.txt"), "w") as fh:
        fh.write(counters(a.tag, a, peak))
    traffic_json(a.tag)
    sass_pages(a.tag)


if __name__ == "__main__":
    main()
