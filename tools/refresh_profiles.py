"""Copy the final-tree evidence of a gpurun (tools/gpu_final.sh +
tools/gpu_ncu_final.sh) into profiles/r02: bench and reference-arm lines,
the C2 launch list, the face capture, per-kernel DRAM traffic
(ncu_traffic.json, read by bench.py's roofline) and the "Final tree"
section of ncu_kernels.md."""
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))
import ncu_profiles as NP  # noqa: E402

G = ROOT / "gpurun_out"
P = ROOT / "profiles" / "r02"
for f in ("ref", "bench"):
    lines = [l for l in (G / "final" / f"{f}.json").read_text().splitlines() if l.startswith("{")]
    (P / f"{f}_final.json").write_text("\n".join(lines) + "\n")
shutil.copy(G / "ncu" / "launches_c2.csv", P / "launches_c2_final.csv")
shutil.copy(G / "ncu" / "c2_face.ncu-rep", P / "ncu_reps" / "c2_face_final.ncu-rep")
tj = P / "ncu_traffic.json"
d = json.loads(tj.read_text())
for key, tag in (("face_flux", "c2_face"), ("recon", "c2_recon_weno"), ("assemble", "c2_assemble_tile"),
                 ("jacobi_sweep", "c2_roe_mf6")):
    r = NP.read(G / "ncu" / f"{tag}.ncu-rep")
    d["c2_n16"][key] = {"kernel": r["name"].strip(), "dram_bytes_per_launch": r.get("rd", 0) + r.get("wr", 0),
                        "read": r.get("rd", 0), "write": r.get("wr", 0),
                        "capture": "end of round 2 (tools/gpu_ncu_final.sh)"}
tj.write_text(json.dumps(d, indent=1) + "\n")
md = P / "ncu_kernels.md"
s = md.read_text()
s = s[:s.index("## Final tree (end of round 2")]
out = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_profiles.py"), str(G / "ncu")], capture_output=True,
                     text=True).stdout
s += ("## Final tree (end of round 2, tools/gpu_ncu_final.sh)\n\nRe-captured on the final tree (pair-batched "
      "Jacobi sweep, tiled assembly, reciprocal / common-denominator combine, three divisions less in the face "
      "kernel, face kernel at 255 registers); same method as above.\n\n" + out[out.index("| capture"):])
md.write_text(s)
print("profiles refreshed")
