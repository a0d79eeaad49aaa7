# the non-headline configurations of BASELINE.json (one gpurun call); lines -> gpurun_out/<tag>_<name>_bench.json
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
Q="--no-cpu-baseline --no-f2 --no-f4"
timeout 900 python bench.py --eps 1e-6 $Q --no-f3 --no-stage3 --no-e2e 2>&1 | tail -1 > gpurun_out/${TAG}_eps_bench.json
timeout 900 python bench.py --workload m120 $Q --no-f3 2>&1 | tail -1 > gpurun_out/${TAG}_m120_bench.json
timeout 1500 python bench.py --workload c2h4 --parents 60000 $Q --no-stage3 --f3-parents 20000 2>&1 | tail -1 > gpurun_out/${TAG}_c2h4_bench.json
timeout 900 python bench.py --workload h2o $Q --no-f3 2>&1 | tail -1 > gpurun_out/${TAG}_h2o_bench.json
for f in gpurun_out/${TAG}_*_bench.json; do echo "$f: $(cut -c1-260 $f)"; done
