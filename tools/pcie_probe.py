"""PCIe probe (development aid): pinned host <-> device copy rates, one direction and both at once,
with 1 or 2 streams per direction, chunked like fks_step_host."""
import torch

GB = 1 << 30
h_in = torch.empty(GB // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(GB // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty(GB // 8, dtype=torch.float64, device="cuda")
d_out = torch.empty(GB // 8, dtype=torch.float64, device="cuda")


def run(streams_per_dir, both, chunks=32, reps=3):
    hs = [torch.cuda.Stream() for _ in range(streams_per_dir)]
    ds = [torch.cuda.Stream() for _ in range(streams_per_dir)]
    n = h_in.numel()
    c = n // chunks
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in hs + ds:
            s.wait_event(e0)
        for i in range(chunks):
            with torch.cuda.stream(hs[i % streams_per_dir]):
                d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
            if both:
                with torch.cuda.stream(ds[i % streams_per_dir]):
                    h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)
        for s in hs + ds:
            e = torch.cuda.Event()
            e.record(s)
            torch.cuda.current_stream().wait_event(e)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for spd in (1, 2, 4):
    t1 = run(spd, False)
    t2 = run(spd, True)
    print(f"{spd} stream(s)/direction: H2D only {1.0 / (t1 * 1e-3):.1f} GiB/s; "
          f"both directions {1.0 / (t2 * 1e-3):.1f} GiB/s each ({t2:.2f} ms per GiB pair)")
