import csv, sys, re
rows=list(csv.reader(open(sys.argv[1])))
# multiple kernels: blocks start with "Kernel Name" rows
i=0
while i < len(rows):
    r=rows[i]
    if r and r[0]=="Kernel Name":
        name=r[1][:70]; hdr=rows[i+1]; i+=2
        ia=hdr.index('Address'); isrc=hdr.index('Source'); iie=hdr.index('Instructions Executed')
        tot=0; calls=[]; prev=None
        while i < len(rows) and rows[i] and rows[i][0]!="Kernel Name":
            rr=rows[i]
            if len(rr)>iie:
                c=int(rr[iie] or 0); tot+=c
                if 'CALL' in rr[isrc] and c: calls.append((rr[isrc].strip()[:40],c))
            i+=1
        print(name, 'total', tot)
        for s,c in calls: print('   ', s, c)
    else: i+=1
