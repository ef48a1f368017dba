mkdir -p gpurun_out/wlab
for spec in base=base m3=build/libgks_minb3.so; do
  tag=${spec%%=*}; lib=${spec#*=}
  if [ "$lib" = "base" ]; then unset GKS_LIB; else export GKS_LIB=$PWD/$lib; fi
  for w in c1 c3 c4 c5; do
    timeout 900 python bench.py --workload $w --no-cpu-baseline --no-converge --no-c5 --steps 5 > gpurun_out/wlab/${tag}_$w.json 2>gpurun_out/wlab/${tag}_$w.err
    python - $tag $w <<'PY'
import json,sys
t,w=sys.argv[1:]
for l in open(f"gpurun_out/wlab/{t}_{w}.json"):
    if l.startswith("{"):
        d=json.loads(l); k=d.get("kernels",{})
        print(t, w, "ms/step %.2f"%d["ms_per_step"], "face %.4f"%k.get("face_flux",{}).get("ms_per_launch",0), flush=True)
PY
  done
done
