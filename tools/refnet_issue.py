"""Host issue time vs device time of the native replication loop
(epi_refnet_run): is the reference-native loop host- or device-bound?"""
import sys, time; sys.path.insert(0, ".")
import torch
from paper_2110_04421_b200.refsim import ReferenceNativeSimulation

for rep in range(4):
    sim = ReferenceNativeSimulation(100_000, base_seed=rep, initial_infections=10, horizon=180)
    counts = torch.zeros((180, 2), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for chunk in (30, 180):
        first = sim.clock
        t0 = time.perf_counter()
        st.record()
        sim.engine.advance_refnet(sim.realizer, first, chunk, counts[first:chunk], sim.records[first:chunk])
        en.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"rep {rep} steps {first}-{chunk}: issue {1e3 * (t1 - t0):.2f} ms, until done {1e3 * (t2 - t0):.2f} ms, "
              f"device {st.elapsed_time(en):.2f} ms", flush=True)
