"""Developer probe: measured FP64 DFMA peak + clocks (not a test)."""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_03121_b200.peaks import measure_fp64_peak  # noqa: E402

samples = []
stop = False


def poll():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True)
        samples.append(r.stdout.strip())
        time.sleep(0.2)


t = threading.Thread(target=poll)
t.start()
print(measure_fp64_peak(reps=20, seconds=4.0))
stop = True
t.join()
print(samples[len(samples) // 2], samples[-3:])
