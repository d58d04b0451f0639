"""HBM ceilings for traffic mixes (torch kernels, CUDA events, best of 10): copy (1R:1W),
write-only (fill), read-only (sum), and 1R:4W (one source copied into four destinations)."""
import json
import torch

n = 1 << 31  # 2 GiB per buffer
a = torch.empty(n, dtype=torch.uint8, device="cuda").fill_(1)
outs = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(4)]


def best(fn, reps=10):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e-3)
    return min(ts)


res = {}
t = best(lambda: outs[0].copy_(a)); res["copy_1R1W_GBps"] = 2 * n / t / 1e9
o64 = outs[0].view(torch.int64)
t = best(lambda: o64.fill_(3)); res["write_only_GBps"] = n / t / 1e9
t = best(lambda: outs[1].zero_()); res["write_only_zero_GBps"] = n / t / 1e9
av = a.view(torch.int64)
t = best(lambda: av.sum()); res["read_only_GBps"] = n / t / 1e9
def four():
    for o in outs:
        o.copy_(a)
t = best(four); res["4x_copy_4R4W_GBps"] = 8 * n / t / 1e9
print(json.dumps(res))
