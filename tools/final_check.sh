# end-of-round check on one GPU box: smoke, the whole GPU suite, the default
# bench line and the NYTimes line (written to gpurun_out/<tag>_*)
tag=${1:-final}; o=gpurun_out; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $o/${tag}_smoke.log)"
timeout 1500 python -m pytest tests -m gpu -q > $o/${tag}_gputests.log 2>&1; echo "gpu tests: $(tail -1 $o/${tag}_gputests.log)"
grep -E "^FAILED|^ERROR" $o/${tag}_gputests.log | head
timeout 900 python bench.py > $o/${tag}_bench_pm.json 2> $o/${tag}_bench_pm.err; echo "bench rc=$?"
timeout 900 python bench.py --workload nytimes --no-cpu-baseline > $o/${tag}_bench_nyt.json 2> $o/${tag}_bench_nyt.err; echo "nyt rc=$?"
for f in $o/${tag}_bench_pm.json $o/${tag}_bench_nyt.json; do python -c "
import json,sys; d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); print('$f'.split('/')[-1], round(d['value']/1e9,3), 'G  e2e', round(d['e2e']['value']/1e9,3), 'frac', round(d['roofline']['frac'],3), d['clocks'])"; done
