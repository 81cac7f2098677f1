# enumeration placement sensitivity (S28 full, S32 2^24 block) after different allocations
python tools/enum_placement.py > gpurun_out/r2s65.log 2>&1
python tools/enum_placement.py >> gpurun_out/r2s65.log 2>&1
