"""Executed-instruction footprint in 128-byte I-cache lines from an ncu source-page CSV:
how many lines cover 50/90/99/... %% of executed instructions, and the no_instruction
stall share on those lines.  usage: python tools/icache_lines.py SOURCE_CSV"""
import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; ix={h:i for i,h in enumerate(hdr)}
data=[]
for r in rows[2:]:
    try: data.append((int(r[ix["Address"]],16), int(r[ix["Instructions Executed"]] or 0), int(r[ix["stall_no_inst"]] or 0), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
    except: pass
lines=collections.defaultdict(lambda:[0,0,0])
for a,n,s,sa in data:
    L=lines[a//128]; L[0]+=n; L[1]+=s; L[2]+=sa
tot=sum(v[0] for v in lines.values()); tni=sum(v[1] for v in lines.values())
srt=sorted(lines.values(), key=lambda v:-v[0])
acc=0; accni=0
marks=[0.5,0.9,0.95,0.99,0.999,0.9999,0.99999]
k=0
print("lines executed:", sum(1 for v in srt if v[0]>0), "=", sum(1 for v in srt if v[0]>0)*128/1024,"KB")
for i,v in enumerate(srt):
    acc+=v[0]; accni+=v[1]
    while k<len(marks) and acc>=marks[k]*tot:
        print(f"{marks[k]*100:.3f}% exec in {i+1} lines = {(i+1)*128/1024:.1f} KB; no_inst on those {100*accni/tni:.1f}%")
        k+=1
# no_inst per line vs exec per line: miss rate proxy
