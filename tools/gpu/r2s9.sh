# retune the fast kernel's knobs after the work elimination changed the work mix
python tools/time_enum.py | sed "s/^/default /"
for t in 8 10 14 16; do TV_SERVICE_THRESH=$t python tools/time_enum.py | sed "s/^/thresh=$t /"; done
for s in 16 24 40; do TV_STACK_S=$s python tools/time_enum.py | sed "s/^/stack=$s /"; done
for th in 256 320; do TV_FAST_THREADS=$th python tools/time_enum.py | sed "s/^/threads=$th /"; done
for c in 128 512; do TV_CTA_SLOTS=$c python tools/time_enum.py | sed "s/^/slots=$c /"; done
TV_ORDER=0 python tools/time_enum.py | sed "s/^/order=0 /"
