"""FP64 DFMA throughput vs resident warps per SM (8 independent chains per
thread): how many warps per SMSP the FP64 pipe needs (csrc/measure.cu)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_28770_b200 import _capi
L = _capi.lib(); dev = torch.device("cuda", 0)
sms = torch.cuda.get_device_properties(0).multi_processor_count
sink = torch.empty(sms * 64, dtype=torch.float64, device=dev)
fl = ctypes.c_double(); st = torch.cuda.current_stream()
for w in (1, 2, 3, 4, 6, 8, 12, 16, 32):
    best = 0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); L.zeus_bench_dfma(sms, 32 * w, 2000, sink.data_ptr(), ctypes.byref(fl), st.cuda_stream); e1.record(); e1.synchronize()
        best = max(best, fl.value / (e0.elapsed_time(e1) / 1e3))
    print(f"warps/SM {w:3d}: {best/1e12:6.2f} TFLOP/s  ({best/1e12/36.7*100:5.1f}% of 36.7)")
