# kernel-only GEMM times (ncu gpu__time_duration, serialized): tools/gemm_ncu.sh M N K [mode]
M=$1; N=$2; K=$3; MODE=${4:-auto}
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv python tools/gemm_time.py $M $N $K $MODE 2>/dev/null \
 | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
h=rows[0]; t=collections.defaultdict(list)
for r in rows[1:]:
    d=dict(zip(h,r))
    if d.get('Metric Name')=='gpu__time_duration.sum': t[d['Kernel Name'][:40]].append(float(d['Metric Value'].replace(',','')))
for k,v in t.items():
    if 'distribution' in k or 'normal' in k: continue
    v=sorted(v); print('$M $N $K', k, 'n=%d median %.2f us'%(len(v), v[len(v)//2]/1000))
"
