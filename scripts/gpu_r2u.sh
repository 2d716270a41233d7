# Does the clocks sampler's start-up perturb the timed region?  Bench with the sampler
# (now started before timing), without it, and with 100 steps, interleaved, same box.
mkdir -p gpurun_out/u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u/build.log 2>&1
s() { python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],4), d.get('clocks'))" $1 $2; }
for i in 1 2; do
  python bench.py --no-cpu-baseline --no-e2e > gpurun_out/u/a.json 2>/dev/null; s gpurun_out/u/a.json clocks_$i
  python bench.py --no-cpu-baseline --no-e2e --no-clocks > gpurun_out/u/b.json 2>/dev/null; s gpurun_out/u/b.json noclocks_$i
  python bench.py --no-cpu-baseline --no-e2e --no-clocks --steps 100 > gpurun_out/u/c.json 2>/dev/null; s gpurun_out/u/c.json noclocks100_$i
  python bench.py --no-cpu-baseline --no-e2e --steps 1000 > gpurun_out/u/d.json 2>/dev/null; s gpurun_out/u/d.json clocks1000_$i
done
