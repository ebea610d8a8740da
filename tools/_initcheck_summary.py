import re,sys,collections
acc=collections.Counter(); other=collections.Counter(); frames={}
cur=None; lines=open(sys.argv[1],errors='replace').read().splitlines()
for i,l in enumerate(lines):
    m=re.search(r'Host API memory access error at host access to (0x[0-9a-f]+) of size (\d+)',l)
    if m:
        cur=(m.group(1),m.group(2)); acc[cur]+=1
        for k in range(i+1,min(i+8,len(lines))):
            if 'Host Frame' in lines[k] and 'cudaMemcpy' not in lines[k] and 'cuMemcpy' not in lines[k]:
                frames.setdefault(cur, lines[k].split('Host Frame:')[1][:160]); break
        continue
    if l.startswith('========= ') and ('Uninitialized' in l or 'Invalid' in l) and 'cudaMemcpy' not in l and 'on access by' not in l:
        other[l[:150]]+=1
for k,v in acc.most_common(30): print(v,k,frames.get(k))
print('other:')
for k,v in other.most_common(30): print(v,k)
