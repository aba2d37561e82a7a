"""Live tensor-pipe peaks used as roofline denominators, with the SM clock sampled during each
loop: kind::i8 (cta_group 1 and 2) and kind::mxf4 (zero and random GF(2)-encoded operands,
short and long loops).  python tools/peaks.py > profiles/r02/peaks.json"""
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1111_6900_b200 import _lib  # noqa: E402


def sampled(fn):
    rows, stop = [], threading.Event()

    def poll():
        while not stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,"
                                      "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                rows.append(out)
            except Exception:
                pass
            time.sleep(0.05)

    t = threading.Thread(target=poll, daemon=True)
    t.start()
    v = fn()
    stop.set()
    t.join(timeout=5)
    return v, rows


torch.cuda.set_device(0)
res = {"gpu": torch.cuda.get_device_name(0)}
for name, fn in [("i8_cta_group1", lambda: _lib.mma_peak(1, 20000)[0]),
                 ("i8_cta_group2", lambda: _lib.mma_peak(2, 20000)[0]),
                 ("mxf4_zero_20k", lambda: _lib.mma_peak_fp4(20000, "zero")),
                 ("mxf4_random_20k", lambda: _lib.mma_peak_fp4(20000, "random")),
                 ("mxf4_random_400k", lambda: _lib.mma_peak_fp4(400000, "random"))]:
    fn()  # warm
    v, rows = sampled(fn)
    res[name] = {"tops": round(v, 1), "smi_samples(sm_mhz,power_w,sw_power_cap)": rows[:8]}
    print(name, round(v, 1), rows[:3], file=sys.stderr)
print(json.dumps(res, indent=1))
