timeout 1500 python tools/scale_model.py C5 1 2 4 8 > gpurun_out/scale_model_C5.json 2> gpurun_out/scale_model_C5.err; echo "model rc=$?"; tail -4 gpurun_out/scale_model_C5.err
python -c "
import json; d=json.load(open('gpurun_out/scale_model_C5.json')); print('t1', d['t1_measured_ms'], {p: (round(v['total_ms'],1), round(v['predicted_efficiency'],3)) for p,v in d['P'].items()})"
timeout 600 python tools/scale_model.py C2 1 2 4 8 > gpurun_out/scale_model_C2.json 2> gpurun_out/scale_model_C2.err; echo "model rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/scale_model_C2.json')); print('t1', d['t1_measured_ms'], {p: (round(v['total_ms'],2), round(v['predicted_efficiency'],3)) for p,v in d['P'].items()})"
