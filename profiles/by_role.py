"""Per-role instruction and stall-sample shares from `ncu --page source --csv --print-source cuda,sass`.
Usage: by_role.py dump.csv warp_attempts
Roles are attributed by CUDA source line (function ranges of kernels_layered.cu, read from the file)."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1]))); wa = float(sys.argv[2])
src = open('paper_1004_0024_b200/csrc/kernels_layered.cu').read().split('\n')
# function start lines
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r'(?:template.*\n)?(?:__device__|__global__|static).*?\b(\w+)\(', l)
    if m and not l.startswith(' '): starts.append((i, m.group(1)))
def func_of(line):
    name = '?'
    for s, n in starts:
        if s <= line: name = n
    return name
role_of = {'producer_warp': 'producer', 'mt_load_operands': 'producer', 'mt_generate8': 'producer',
           'post_warp': 'post', 'far_warp': 'far', 'far_update': 'sweep', 'attempt': 'sweep', 'feed': 'sweep',
           'sweep_warp': 'sweep', 'wait_post': 'sweep', 'layer_transition': 'transition'}
fname = None; hdr = None
inst = collections.Counter(); samp = collections.Counter(); stall = collections.defaultdict(collections.Counter)
for r in rows:
    if not r: continue
    if r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; ix = {h: i for i, h in enumerate(hdr)}; continue
    if hdr is None or len(r) != len(hdr) or not r[0].isdigit(): continue
    line = int(r[0])
    if fname == 'kernels_layered.cu':
        f = func_of(line); role = role_of.get(f, f)
    elif fname == 'device_mt.cuh': role = 'producer'
    elif fname == 'device_math.cuh':
        role = 'producer' if line < 40 else 'sweep'   # mt_recurrence/temper/u32_to_unit vs exp kinds
    else: role = fname
    i_sm = hdr.index('# Samples'); i_in = hdr.index('Instructions Executed')
    inst[role] += int(r[i_in]); samp[role] += int(r[i_sm])
    for h in hdr:
        if h.startswith('stall_') and 'Not Issued' not in h: stall[role][h[6:]] += int(r[ix[h]] or 0)
tot = sum(samp.values())
for role in sorted(inst, key=lambda k: -inst[k]):
    top = ', '.join(f'{k} {100*v/max(1,samp[role]):.0f}%' for k, v in stall[role].most_common(5))
    print(f'{role:12s} inst/warp-attempt {inst[role]/wa:7.1f}   samples {100*samp[role]/tot:5.1f}%   {top}')
print('total inst/warp-attempt', round(sum(inst.values()) / wa, 1))
