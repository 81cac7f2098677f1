"""Device time of all 2^32 S^{32}_{3,8} genomes in one enumeration call (CUDA events), checked
against the oracle's full-space tallies.  Development aid (slice-size A/B via TV_SLICE_LOG2)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2205_15311_b200 import classify as C
from paper_2205_15311_b200.genome import space_from_preset
dh = C.DeviceHistogram((7,), 7, C.shape_words_for(19), 1 << 21)
sp = space_from_preset("s32_3_8")
dh.enumerate_range(sp, 0, 1 << 24, 19, 0, True)  # warm-up
dh.clear()
s = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
dh.enumerate_range(sp, 0, 1 << 32, 19, 0, True)
e1.record(s)
torch.cuda.synchronize()
gold = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                                   "hist_s32_full.json")))
h = dh.export()
print(f"slice 2^{os.environ.get('TV_SLICE_LOG2', '26')}: {e0.elapsed_time(e1):.1f} ms, "
      f"tallies ok {h.tallies.tolist() == gold['tallies']}, keys {len(h)} (gold {gold['n_keys']})", flush=True)
