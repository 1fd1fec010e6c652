timeout 300 python tools/cublas_f32out.py 16384 40 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 12 --csv python tools/cublas_f32out.py 16384 1 2>/dev/null | grep -v "^==" | python -c "
import sys,csv
rows=list(csv.reader(sys.stdin))
h=None
for r in rows:
    if len(r)>5 and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); print(d['ID'], d['Kernel Name'][:70], d['Grid Size'], d['Cluster Size'] if 'Cluster Size' in d else '', d['Metric Name'], d['Metric Value'])
"
