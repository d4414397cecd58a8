timeout 600 python tools/time_fs.py c5pl 4 5 2>&1 | tail -1
timeout 600 python tools/profile_step.py c5pl 4 auto 2 > gpurun_out/plain_c5pl.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "search/" --csv --log-file gpurun_out/launch_c5pl.csv python tools/profile_step.py c5pl 4 auto 2 > /dev/null 2>&1
python3 - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/launch_c5pl.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
hdr=rows[hi]; ik=hdr.index('Kernel Name'); iv=hdr.index('Metric Value')
for r in rows[hi+1:]: print(round(float(r[iv].replace(',',''))/1e3,1), 'us', r[ik][:70])
P
