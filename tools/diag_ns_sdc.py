import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, ctypes as C
from oracle import oracle as O
import paper_1309_7327_b200 as P
from paper_1309_7327_b200 import workloads as W
from test_gpu_ns_steppers import acoustic_dt, _cb
n=12; DX=1e-4
T,p,uvw,Y=W.ns_primitives(n); U0=O.ns_conserved(T,p,uvw,Y)
dt=acoustic_dt((T,p,uvw,Y),DX)
g=dict(np.load('tests/golden/golden.npz'))
r1=O.ns_rhs(U0,DX,0); op=P.NsOperator(n,n,n,DX); r2=op.full(0.0,U0)
print("single rhs", ["%.1e"%(np.abs(r2[v]-r1[v]).max()/np.abs(r1[v]).max()) for v in range(14)])
for steps in (1,2,5,10):
    cb=_cb(n,0); u0=U0.ravel().copy(); uo=np.empty_like(u0); res=np.zeros(64); sw,fe,es=C.c_int(),C.c_int(),C.c_int()
    O.lib().or_integrate_sdc(cb,None,u0.size,O.dp(u0),C.c_double(0),C.c_double(steps*dt),steps,2,O.dp(g['nodes_gl3']),O.dp(g['q_gl3']),O.dp(g['s_gl3']),4,C.c_double(0),1,O.dp(uo),O.dp(res),64,C.byref(sw),C.byref(fe),C.byref(es))
    ref=uo.reshape(U0.shape)
    st=P.SdcStepper(3,P.StepControls(4,0.0)); got,d=st.integrate(op.full,U0,0.0,steps*dt,steps)
    print(steps, ["%.1e"%(np.abs(got[v]-ref[v]).max()/np.abs(ref[v]).max()) for v in range(14)])
    print("   change/step", ["%.1e"%(np.abs(ref[v]-U0[v]).max()/np.abs(ref[v]).max()) for v in range(14)])
