import numpy as np, time
n=10_500_000
g=np.random.rand(n); f=np.empty(n,np.float32); d=np.empty(n)
for name,fn in (("convert f64->f32",lambda: np.copyto(f,g,casting='unsafe')),("copy f64",lambda: np.copyto(d,g))):
    fn(); t=time.perf_counter()
    for _ in range(10): fn()
    dt=(time.perf_counter()-t)/10
    print(f"1 thread {name}: {dt*1e3:.2f} ms")
