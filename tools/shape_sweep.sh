# persistent-launch CASPS over worlds x launch shapes (bench.py --shape)
WS=${WS:-"296 512 1024 2048"}
SHAPES=${SHAPES:-"8x2 4x4"}
for W in $WS; do for sh in $SHAPES; do
 printf "W=$W shape=$sh "; timeout 120 python bench.py --worlds $W --shape $sh --no-cpu --no-c5 --e2e-steps 3 --steps 96 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), 'M CASPS', round(d['roofline']['kernel_ms_per_tick']*1e3,1), 'us/tick')"
done; done
