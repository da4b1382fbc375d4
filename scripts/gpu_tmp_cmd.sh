rm -f /tmp/ts.bin
CVB_TC_DEBUG=16 CVB_TC_TS_FILE=/tmp/ts.bin timeout 300 python bench.py --steps 1 --warmup 0 --no-graph --no-cpu-baseline --no-e2e --no-compare > gpurun_out/tl.json 2> gpurun_out/tl.err; echo rc $?
cp /tmp/ts.bin gpurun_out/ts.bin; ls -la gpurun_out/ts.bin
python scripts/dbg/timeline.py gpurun_out/ts.bin
