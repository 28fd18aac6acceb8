import time, numpy as np, oracle, os
oracle.build()
print("threads", oracle.num_threads())
for cfg,(n,k,g,s) in {2:(10**6,10,3.0,2),3:(10**7,100,3.0,3),4:(10**6,32,2.2,4)}.items():
    a=oracle.alpha(g); R=oracle.target_radius(n,k,a)
    t0=time.perf_counter(); th,r=oracle.sample_points(n,a,R,s); t1=time.perf_counter()
    m,t=oracle.sweep_count(th,r,R,0,n); t2=time.perf_counter()
    print(cfg,"sample",t1-t0,"sort+sweep",t2-t1,"m",m,"tests",t, flush=True)
n=10**8; a=oracle.alpha(2.7); R=oracle.target_radius(n,16,a)
t0=time.perf_counter(); th,r=oracle.sample_points(n,a,R,5); t1=time.perf_counter()
print("cfg5 sample", t1-t0, flush=True)
q=np.arange(16,dtype=np.uint32)
t0=time.perf_counter(); off,nbr,nt=oracle.rows(th,r,R,q); t1=time.perf_counter()
print("cfg5 rows 16", t1-t0, off[-1], flush=True)
