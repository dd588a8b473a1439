import csv,sys
for cz in sys.argv[1:]:
    rows=list(csv.reader(open(f'/root/repo/gpurun_out/cz_{cz}.csv')))
    hdr=next(i for i,r in enumerate(rows) if 'Kernel Name' in r); h=rows[hdr]
    ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
    d={}
    for r in rows[hdr+1:]:
        if ', 0, 2>' in r[ki] or ', 2, 2>' in r[ki] or ', 3, 2>' in r[ki]: d.setdefault(r[ii],{})[r[mi]]=float(r[vi].replace(',',''))
    v=list(d.values())[0]
    t=v['gpu__time_duration.sum']; rd=v['dram__bytes_read.sum']; wr=v['dram__bytes_write.sum']
    print(f"cz={cz:5s} grid={int(v.get('launch__grid_size',0)):5d} {t/1e3:8.1f}us rd {rd/1e9:.2f}GB wr {wr/1e9:.2f}GB  {(rd+wr)/t:.0f} GB/s  B/pt {(rd+wr)/1.0077e9:.2f}")
