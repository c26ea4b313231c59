"""Write profiles/ncu_traffic.json from an ncu --set full report: DRAM bytes per launch of
K1-K4 and each kernel's L1 data-pipe (LSU wavefront) utilisation, the limiter of K2/K3."""
import csv
import json
import subprocess
import sys
from pathlib import Path

rep = sys.argv[1]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}
out = {}
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')]
    tot = 0.0
    for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum'):
        i = hdr.index(k)
        tot += float(r[i].replace(',', '')) * scale[units[i]]
    key = ('K2_forward_dual' if 'fwd_kernel' in name else 'K3_adjoint' if 'adj_kernel' in name
           else 'K1_prox_warp' if 'pack_kernel' in name else 'K4_adjoint_update'
           if 'update_kernel' in name else name)
    out[key] = tot
    i = hdr.index('l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed')
    out.setdefault('l1_data_pipe_frac', {})[key] = float(r[i].replace(',', '')) / 100.0
out['source'] = Path(rep).name + ' (C3, 20-item PDHG launch, ncu --set full --clock-control none)'
Path('profiles').mkdir(exist_ok=True)
Path('profiles/ncu_traffic.json').write_text(json.dumps(out, indent=1) + '\n')
print(out)
