import sys, numpy as np, torch
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import paper_2603_27914_b200 as P
from paper_2603_27914_b200 import _lib
from oracle import itq3_oracle as O
lib=_lib.load()
g=torch.Generator(device='cuda'); g.manual_seed(1)
rows, cols, M = 128, 256, 16
w=torch.randn((rows,cols),generator=g,device='cuda')/16
q=P.quantize_tensor(w)
X=torch.randn((cols,M),generator=g,device='cuda')
BN=16; N=32
act=torch.empty(lib.itq3_mmq8_act_nbytes(cols,M),dtype=torch.uint8,device='cuda')
_lib.call("itq3_rotate_act_i8", _lib.ptr(X), _lib.F32, cols, M, X.stride(0), X.stride(1), _lib.ptr(act), None, _lib.stream_ptr(X.device))
a=act.cpu().numpy()
def sw(n,c): return (n>>3)*1024+(n&7)*128+((c^(n&7))<<4)
Bt=np.zeros((N,256),np.int64)
for n in range(N):
    for e in range(256):
        kb=e&127
        Bt[n,e]=np.int8(a[(e>>7)*(N*128)+sw(n,kb>>4)+(kb&15)])
meta=a[512*BN:512*BN+8*BN].view(np.float32).reshape(BN,2)
Xn=X.cpu().numpy().astype(np.float64)
H=O.hadamard(256)
for m in range(3):
    qv=Bt[m]+256*Bt[BN+m]
    xr=H@Xn[:,m]   # unnormalized
    f=meta[m,0]*16
    print('tok',m,'max|x_r - q*2^ex|',np.max(np.abs(xr-qv*f)), 'scale',f, 'Q ok', abs(meta[m,1]-qv.sum()*meta[m,0]))
wr=q.mmq8_layout().cpu().numpy()
pay=q.payload().cpu().numpy()
quants,sb,zb,_=O.split_payload(pay,256,False)
codes,_=O.unpack_planes(quants,256)
c=(codes+1)
bad=0
for r in range(rows):
    for B in range(64):
        byte=wr[(B>>4)*2048+r*16+(B&15)]
        exp=sum(int(c[r,64*i+B])<<(2*i) for i in range(4))
        bad+= byte!=exp
print('repack bad bytes',bad, 'scale ok', np.all(wr[8192:8448].view(np.uint16)==sb))
Y=torch.empty((rows,M),dtype=torch.float32,device='cuda')
_lib.call("itq3_mmq8", _lib.ptr(q.mmq8_layout()), rows, cols, _lib.ptr(act), M, _lib.ptr(Y), _lib.F32, Y.stride(0), Y.stride(1), None, _lib.stream_ptr(X.device))
Yn=Y.cpu().numpy()
d=O.f16_value(sb)
D=c.astype(np.int64)@Bt.T   # rows x N
emu=np.zeros((rows,M))
for m in range(M):
    v=D[:,m]+256*D[:,BN+m]
    emu[:,m]=d*(meta[m,0]*v-1*meta[m,1])
exact=O.dequantize(pay,rows,cols,256,False)@Xn
print('emu vs exact',np.max(np.abs(emu-exact)),'gpu vs emu',np.max(np.abs(Yn-emu)))
print(Yn[:3,:3]); print(emu[:3,:3])
# hypothesis checks: gpu D from Y
Dg=np.zeros_like(emu)
for m in range(M):
    Dg[:,m]=(Yn[:,m]/d+meta[m,1])/meta[m,0]
print('Dg',Dg[:2,:4]); print('D0+256D1',(D[:,:BN]+256*D[:,BN:])[:2,:4])
print('D0 only',D[:2,:4],'D1',D[:2,BN:BN+4])
