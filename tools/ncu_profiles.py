"""Summarise the per-kernel ncu --set full captures of tools/gpu_ncu_all.sh
into profiles/r02/ncu_kernels.md: measured duration, ncu DRAM bytes,
algorithmic bytes (or FP64 flops) per launch from the workload sizes, and
the fraction of the HBM / FP64 peak.

    python tools/ncu_profiles.py gpurun_out/ncu > profiles/r02/ncu_kernels.md
"""
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
HBM = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
    else 6548.2
FP64 = 33.77  # live DFMA probe (gks_fp64_peak) on this pool, TFLOP/s

# workload sizes (bench.py config / gks_handle_info), C2 and C3: sphere n=16; C1: box n=16
C2 = dict(nc=1474560, nf=2955264, nfq=8865792)
C2["nfi"] = C2["nf"] - 6 * 16 * 16 * 4 * 2  # interior faces: two spherical shells of boundary faces
C1 = dict(nc=6 * 16 ** 3)
# C1 n=64 periodic box (Roe GMRES): 4 faces per tet shared -> 2 nc interior faces, nnz = 4 nc
_n1 = 6 * 64 ** 3
C1B = {"spmv": _n1 * (4 + 4 * 8 + 2 * 40 + 40 + 40 + 200 + 40 + 40) + _n1 * (200 + 40)}
K, M, S = 13, 4, 6  # padded WENO record of the sphere (k_recon_weno<13, 4, 6>)
HA, HG, HM = 4, 5, 4  # padded HWENO record (k_recon_hweno<4, 5, 4>)


def model():
    nc, nfq, nfi = C2["nc"], C2["nfq"], C2["nfi"]
    n5 = 5 * nc
    nnz = 2 * nfi
    per_row = nnz / nc
    faces = nfi / nc
    sweep = nc * (4 + per_row * 8 + faces * 40 + 40 + 40 + 200 + 40 + 40)
    return {
        "c2_recon_weno": ("bytes", nc * (9 * K * 8 + K * 4 + M * 3 * S * 8 + M * S * 4 + M + 360 + 40 + 360),
                          "operator records + Q gathers (40 B/cell, neighbours cached) + C write"),
        "c3_recon_hweno": ("bytes", nc * (9 * (HA + 3 * HG) * 8 + (HA + HG) * 4 + HG * 8 + 360 + 40 + 120 + 360),
                           "operator records (linear weights: no sub-stencils) + Q, grad + C write"),
        "c2_assemble5": ("bytes", nfq * 40 + nc * 44 + 2 * nfq * 4, "contributions + CSR list + res write"),
        "c2_assemble_tile": ("bytes", nfq * 40 + nc * 44 + 2 * nfq * 4, "contributions + CSR list + res write"),
        "c1_roe_mf5": ("bytes", C1B["spmv"], "C1 n=64: CSR + face records + prims + x + D + D^-1 + out (+pre)"),
        "c2_roe_mf6": ("bytes", sweep, "CSR + face records + prims + x + D^-1 + b + out"),
        "c2_axpy_dot": ("bytes", 4 * 8 * n5, "w read+write, v_i, v_(i+1)"),
        "c2_dot2": ("bytes", 2 * 8 * n5, "w (twice, one pass) and v_0"),
        "c2_jac_faces": ("bytes", nfi * (8 + 2 * 40 + 32 + 2 * 200 + 40), "Q of both cells, geometry, 2 blocks"),
        "c2_jac_diag": ("bytes", nc * (4 + 40 + 8 + 8 + 400) + nnz * 56, "D, D^-1 write + face lists"),
        "c2_face": ("flops", nfq * (4648 + 720), "reference-model FP64 ops per face point (SURVEY 8d)"),
        "c3_face11": ("flops", nfq * (4648 + 720 + 1239), "+ point value (compact)"),
        "c1_gm_arnoldi": ("latency", None, "one Arnoldi column of a 24,576-cell system in one cluster kernel"),
    }


KEYS = {"dur": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
        "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "warps": "sm__warps_active.avg.pct_of_peak_sustained_active", "regs": "launch__registers_per_thread",
        "dramp": "dram__throughput.avg.pct_of_peak_sustained_elapsed"}
SCALE = {"ns": 1e-9, "nsecond": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def read(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, r = rows[0], rows[1], rows[2]
    out = {"name": re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).replace("void ", "").replace("gks::", "")}
    for k, m in KEYS.items():
        if m in hdr:
            v = float(r[hdr.index(m)].replace(",", ""))
            out[k] = v * SCALE.get(units[hdr.index(m)], 1)
    stalls = []
    for i, h in enumerate(hdr):
        mm = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio", h)
        if mm and r[i]:
            stalls.append((float(r[i]), mm.group(1)))
    out["stalls"] = ", ".join(f"{n} {v:.1f}" for v, n in sorted(stalls, reverse=True)[:3])
    return out


def main(d):
    d = Path(d)
    mdl = model()
    print("# Per-kernel ncu captures (round 2)\n")
    print("`ncu --set full --clock-control none`, one launch of each kernel in `python bench.py --steps 1 "
          "--warmup 1` (tools/gpu_ncu_all.sh).  ncu replays serialise the launch and flush caches, so "
          "durations are cold-cache upper bounds; the bench's in-step CUDA-event timings are the headline.  "
          f"achieved = algorithmic bytes (flops) / ncu duration; peaks: HBM {HBM} GB/s (MEASURED_PEAKS.json), "
          f"FP64 {FP64} TF/s (live DFMA probe).\n")
    print("| capture | kernel | ncu duration | algorithmic / launch | achieved | frac of peak | DRAM read+write "
          "(ncu) | DRAM / algorithmic | FP64 pipe | warps active | regs | top stalls (cyc/issue) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for tag, (kind, amount, what) in mdl.items():
        rep = d / f"{tag}.ncu-rep"
        if not rep.exists():
            continue
        r = read(rep)
        dur = r["dur"]
        dram = r.get("rd", 0) + r.get("wr", 0)
        if kind == "bytes":
            ach = amount / dur / 1e9
            col = (f"{amount / 1e6:.1f} MB ({what})", f"{ach:.0f} GB/s", f"{ach / HBM:.2f} HBM",
                   f"{dram / amount:.2f}")
        elif kind == "flops":
            ach = amount / dur / 1e12
            col = (f"{amount / 1e9:.2f} GFLOP ({what})", f"{ach:.2f} TF/s", f"{ach / FP64:.2f} FP64", "-")
        else:
            col = (what, "-", "-", "-")
        print(f"| {tag} | {r['name']} | {dur * 1e3:.4f} ms | {col[0]} | {col[1]} | {col[2]} | {dram / 1e6:.1f} MB | "
              f"{col[3]} | {r.get('fp64', 0):.1f}% | {r.get('warps', 0):.1f}% | {int(r.get('regs', 0))} | "
              f"{r['stalls']} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ncu")
