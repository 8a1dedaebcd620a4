set -u
O=gpurun_out/r02b; mkdir -p $O
PERMB200_TOL_REPORT=$O/tol_report.json timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_runner.py tests/test_gpu_plain.py tests/test_gpu_dd.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" > $O/status.txt
timeout 300 python tools/m5_run.py --alg ryser --workload M3 --ledger-in /nonexistent --out $O/m3r --budget-s 600 --max-segments 5 --segment-units 64 > $O/m3r1.log 2>&1; echo "m3r1 rc=$?" >> $O/status.txt
mkdir -p /tmp/m3r_in && cp $O/m3r/*.npz $O/m3r/*.csv /tmp/m3r_in/
timeout 300 python tools/m5_run.py --alg ryser --workload M3 --ledger-in /tmp/m3r_in --out $O/m3r2 --budget-s 600 --segment-units 64 > $O/m3r2.log 2>&1; echo "m3r2 rc=$?" >> $O/status.txt
python -c "
import sys; sys.path.insert(0,'.')
import json, torch, synth, paper_1606_05836_b200 as pb
A=torch.from_numpy(synth.workload('M3')).cuda()
v=complex(pb.ryser(A).item()); s=json.load(open('$O/m3r2/m5_status.json'))
print('one-shot', v, 'resumed', s.get('value'), 'equal', s.get('value')==[v.real,v.imag])" > $O/m3r_check.log 2>&1
