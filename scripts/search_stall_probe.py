"""Repeated d_r searches at cfg4 with CPU time and context switches per call: host stalls inside
the driver show up as wall time without CPU time (STGP_POOL=0 to compare)."""
import os, sys, time, resource, threading
sys.path.insert(0, ".")
import paper_2602_03609_b200 as S
theta = S.synth.THETA_T3
x, y, t, resp = S.synth.station_day(10000, 110, box=(4.6e6, 2.9e6), theta=theta, seed=20260203)
perm = S.order_observations_perm(t, 20260203)
x, y, t, resp = x[perm], y[perm], t[perm], resp[perm]
print("nproc", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "load", open("/proc/loadavg").read().strip(), flush=True)
ctx = S.Context(0)
ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
ind = S.sts_kmeanspp(ds, 1000, 20260203)
print("threads", threading.active_count(), len(os.listdir("/proc/self/task")), flush=True)
for rep in range(int(os.environ.get("REPS", "8"))):
    r0 = resource.getrusage(resource.RUSAGE_SELF); c0 = time.process_time()
    t0 = time.perf_counter(); nb = S.residual_neighbors(ds, theta, ind, 30); dt = time.perf_counter() - t0
    r1 = resource.getrusage(resource.RUSAGE_SELF); c1 = time.process_time()
    print(f"search {rep}: wall {dt:.3f}s cpu {c1-c0:.3f}s nivcsw {r1.ru_nivcsw-r0.ru_nivcsw} nvcsw {r1.ru_nvcsw-r0.ru_nvcsw} minflt {r1.ru_minflt-r0.ru_minflt} majflt {r1.ru_majflt-r0.ru_majflt} load {open('/proc/loadavg').read().split()[:3]}", flush=True)
    del nb
