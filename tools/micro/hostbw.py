import numpy as np, time, os, threading
n = 180 << 20
src = np.ones(n, np.uint8); dst = np.zeros(n, np.uint8)
print("cpus", len(os.sched_getaffinity(0)), os.cpu_count())
for T in (1, 4, 8, 16, 32):
    if T > len(os.sched_getaffinity(0)): break
    chunks = np.array_split(np.arange(n, dtype=np.int64)[::1 << 20], T)
    def work(i):
        a = (n * i) // T; b = (n * (i + 1)) // T
        np.copyto(dst[a:b], src[a:b])
    for rep in range(3):
        th = [threading.Thread(target=work, args=(i,)) for i in range(T)]
        t0 = time.perf_counter(); [t.start() for t in th]; [t.join() for t in th]; dt = time.perf_counter() - t0
    print(T, "threads", round(n / dt / 1e9, 1), "GB/s copy (read+write = 2x)")
