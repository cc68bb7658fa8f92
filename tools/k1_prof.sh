# usage: bash /tmp/k1prof.sh TAG "cfgs"
TAG=$1; CF=${2:-"2 4 5"}
for c in $CF; do ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active -k regex:"corner|enclose_kernel" -c 3 --csv python tools/profile_step.py $c > gpurun_out/${TAG}_k1_$c.csv 2>&1; done
python - "$TAG" $CF <<'PY'
import csv,io,sys
tag=sys.argv[1]
for c in sys.argv[2:]:
    txt=open(f"gpurun_out/{tag}_k1_{c}.csv").read()
    i=txt.find("\"ID\"")
    rows=list(csv.DictReader(io.StringIO(txt[i:])))
    for r in rows:
        n=r["Metric Name"].split("__")[1][:22]
        print(c, r["Kernel Name"][:36], n, r["Metric Value"])
PY
