"""Host cost of the torch calls on the per-solve path (A/B tool)."""
import time, torch
h = torch.zeros((1024,1024)).pin_memory()
d = torch.empty((1024,1024), device="cuda")
cs = torch.cuda.Stream()
def t(name, fn, n=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(n): fn()
    dt=(time.perf_counter()-t0)/n*1e6
    torch.cuda.synchronize()
    print(f"{name:40s} {dt:6.2f} us")
t("is_pinned", lambda: h.is_pinned())
def ctx():
    with torch.cuda.stream(cs): pass
t("stream ctx", ctx)
t("Event()", lambda: torch.cuda.Event())
e=torch.cuda.Event()
t("event.record(cs)", lambda: e.record(cs))
t("h.to(cuda, nb)", lambda: h.to("cuda", non_blocking=True))
t("d.copy_(h, nb)", lambda: d.copy_(h, non_blocking=True))
t("current_stream()", lambda: torch.cuda.current_stream())
t("cur.wait_event(e)", lambda: torch.cuda.current_stream().wait_event(e))
t("d.record_stream(cs)", lambda: d.record_stream(cs))
t("torch.device('cuda')", lambda: torch.device("cuda"))
t("torch.empty cuda", lambda: torch.empty((1024,1024), device="cuda"))
t("h.numpy()", lambda: h.numpy())
