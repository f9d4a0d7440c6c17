"""Config-5 leg of bench.py alone (diagnostics): reference.json sweep, decompose.json sweep, 5x8 scale."""
import sys, json, time
sys.argv=['bench.py']
import importlib.util
spec=importlib.util.spec_from_file_location('bench','/root/repo/bench.py'); b=importlib.util.module_from_spec(spec); spec.loader.exec_module(b)
t=time.time()
r=b.run_config5()
print(time.time()-t, r['traces_identical'])
print(json.dumps([(p['rate'], p['trace_identical'], p['reference']['rounds'], p['gpu']['rounds_per_s'], p['reference']['rounds_per_s']) for p in r['decompose']['points']]))
