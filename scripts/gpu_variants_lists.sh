#!/bin/bash
# per-kernel times (ncu launch list, last real launches) of the list kernels for each library variant
mkdir -p gpurun_out
TAG=${TAG:-r2v}
for v in "$@"; do
  lib=$PWD/paper_2301_06984_b200/_lib/var_$v.so
  [ "$v" = base ] && lib=$PWD/paper_2301_06984_b200/_lib/libabsim_gpu.so
  ABSIM_GPU_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_$v.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${TAG}_$v.log 2>&1
  python - <<PY
import csv,re,statistics
rows=[r for r in csv.reader(open("gpurun_out/${TAG}_$v.csv")) if len(r)>10]
h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
d={}
for r in rows[1:]:
    name=re.split(r"[(<]", re.sub(r"^void ","",r[ki]).replace("<unnamed>::",""))[0]
    t=float(r[vi].replace(",",""))/1e6
    if t>0.2: d.setdefault(name,[]).append(t)
print("$v", " ".join("%s=%.2f(x%d)"%(k.replace("k_",""),statistics.median(v),len(v)) for k,v in d.items() if k.startswith("k_list") or k=="k_force"))
PY
  rm -f gpurun_out/${TAG}_$v.csv
done
