TV_TAIL_PROF=1 python tools/time_s32.py
