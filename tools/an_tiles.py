import numpy as np,sys
raw=np.fromfile(sys.argv[1],dtype=np.uint64)
it=raw[65536*8:].reshape(4,512,16).astype(np.int64)
d=it[0]
base=d[100,8]
print("gn g  Kld  Vld  Sissue Sseen  Parr  MMA:preV postV PVissue")
for gn in range(100,112):
    g=gn&1
    print(gn,g,*[d[gn,k]-base for k in (15,14,9,4*g,4*g+3,10,11,8)])
x=np.arange(20,400)
print("median V wait (postV-preV)", np.median(d[x,11]-d[x,10]), " P wait (PVissue-postV)", np.median(d[x,8]-d[x,11]))
print("median V load issue -> PV issue", np.median(d[x,8]-d[x,14]), " K load -> S issue", np.median(d[x,9]-d[x,15]))
