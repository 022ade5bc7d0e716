timeout 1800 python tools/scale_model.py C5 1 2 4 8 > gpurun_out/scale_model_C5.json 2> gpurun_out/scale_model_C5.err; echo "model rc=$?"; tail -5 gpurun_out/scale_model_C5.err
python -c "
import json; d=json.load(open('gpurun_out/scale_model_C5.json')); print('t1', d['t1_measured_ms'], {p: (round(v['total_ms'],1), round(v['predicted_efficiency'],3)) for p,v in d['P'].items()}); print(d.get('alt_interior_dist_gepp_ms'))"
