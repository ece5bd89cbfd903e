"""Host-path (C ABI bed_forward_host_f32) timing for several chunk sizes (dev tool)."""
import os
import subprocess
import sys
import time

if len(sys.argv) > 1:
    import torch

    sys.path.insert(0, ".")
    import paper_2207_04228_b200 as bed
    from paper_2207_04228_b200 import _native, datagen

    n, batch = 4, 1 << 22
    a = datagen.gen_spd_device(batch, n, 7).cpu().pin_memory()
    lam = torch.empty((batch, n)).pin_memory()
    vec = torch.empty((batch, n, n)).pin_memory()
    st = torch.empty((batch,), dtype=torch.int32).pin_memory()
    cfg = _native.make_config(bed.SolverConfig(deflation_tol=3e-12, max_double_steps=16), n)
    call = lambda: _native.forward_host_f32(a.data_ptr(), batch, n, lam.data_ptr(), vec.data_ptr(),  # noqa: E731
                                            st.data_ptr(), None, cfg, 0)
    call()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    print(f"chunk {os.environ.get('BED_HOST_CHUNK_MB', '64')} MB: {batch / min(ts) / 1e6:.1f} M/s")
else:
    for mb in ("4", "8", "16", "32", "64"):
        subprocess.run([sys.executable, __file__, "run"], env={**os.environ, "BED_HOST_CHUNK_MB": mb})
