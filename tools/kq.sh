python -c "
import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], round(d['ms_per_step'],2), d['iterations'], {k:round(v['ms']*1e3,1) for k,v in d['kernels'].items()}, round(d['e2e']['ms_per_step'],2))" $1
