"""Aggregate a tools/ncu_lines.py table (all lines) of a place kernel into phases,
using marker comments of gt_v3.cuh: python tools/phase_lines.py k_p1|k_p2|k_p3 table.txt"""
import re, sys
kern, f = sys.argv[1], sys.argv[2]
src = open('paper_2501_06872_b200/csrc/gt_v3.cuh').read().split('\n')
def find(s, start=0):
    for i in range(start, len(src)):
        if s in src[i]:
            return i + 1
    raise KeyError(s)
rows = []
head = None
for l in open(f):
    if l.startswith('instr='):
        head = l.strip()
    m = re.match(r'(\S+)\s*:(\d+)\s+ins\s+([\d.]+)% stall\s+([\d.]+)% bank\s+([\d.]+)%\s+(.*)', l)
    if m:
        rows.append((m.group(1), int(m.group(2)), float(m.group(3)), float(m.group(4)), float(m.group(5)), m.group(6)))
if kern == 'k_p1':
    k = find('k_p1(const P1Args a) {')
    marks = [('setup', k), ('tile setup/wait', find('for (int j = 0; j < nplace; ++j) {', k)), ('marks', find('// mark the first item of every non-empty', k)),
             ('rank', find('__syncthreads();  // (A) tile landed', k)), ('scan+epi', find('__syncthreads();  // (B) ranks done', k)),
             ('seg_hi', find('// source-high boundaries inside this tile', k)), ('stage', find('// stage payloads and global indices by digit', k)),
             ('writeout', find('__syncthreads();  // (C)', k)), ('zero+end', find('if constexpr (kFast) {\n'.split('\n')[0], find('const uint32_t nout = kSlab', k) + 12)),
             ('END', find('// -------------------------------------------------- record passes', k))]
elif kern == 'k_p2':
    k = find('__global__ void __launch_bounds__(WW * 32, kMinB) k_p2(')
    marks = [('setup', k), ('tile setup', find('for (uint32_t g = blockIdx.x; g < ntall; g += gridDim.x) {', k)), ('place setup/wait', find('for (int jj = 0; jj < nplace; ++jj) {', k)),
             ('rank', find('__syncthreads();  // (A)', k)), ('scan+epi', find('__syncthreads();  // (B)', k)), ('stage', find('tick(3);', k)),
             ('writeout', find('__syncthreads();  // (C)', k)), ('zero+end', find('if constexpr (kFast) zero_s<T2_>', k)), ('END', find('// ---------------------------------------------------------------- L3 units', k))]
else:
    k = find('k_p3(const P3Args a) {')
    marks = [('setup', k), ('unit setup/wait', find('for (int it = 0;; ++it) {', k)), ('rank', find('__syncthreads();  // (A)', k)), ('scan+offsets', find('__syncthreads();  // (B)', k)),
             ('stage', find('const uint32_t oo = align_items_u32(t_e);', k)), ('store', find('__syncthreads();  // (C)', k)), ('zero+end', find('if constexpr (kFast) zero_s<TT>', k)),
             ('END', find('// ---------------------------------------------------------------- planning', k))]
helpers = {'flat_scan_fast': (find('__device__ __forceinline__ void flat_scan_fast'), find('// In-place exclusive scan of a[0..n)')),
           'flat_bases (generic)': (find('__device__ __forceinline__ void flat_bases_epi'), find('// flat_bases_epi\'s scan on 32-bit shared')),
           'zero_u32': (find('__device__ __forceinline__ void zero_u32'), find('__device__ __forceinline__ void zero_u32') + 4)}
agg = {}
for fn, ln, i, s, b, t in rows:
    name = 'other'
    if fn.startswith('gt_v3.cuh'):
        for (nm, lo), (_, hi) in zip(marks, marks[1:]):
            if lo <= ln < hi:
                name = nm
                break
        else:
            for nm, (lo, hi) in helpers.items():
                if lo <= ln < hi:
                    name = nm
    elif fn.startswith('gt_common'):
        name = 'gt_common (accessors, mbarrier wait)'
    a = agg.setdefault(name, [0.0, 0.0])
    a[0] += i
    a[1] += s
print(head)
m = re.match(r'instr=(\d+)', head)
per_slot = int(m.group(1)) / (2 ** 29 / 32) if m else 0
for nm, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f'{nm:40s} ins {v[0]:5.1f}% (~{v[0] * per_slot / 100:5.1f}/slot if E records)  stall {v[1]:5.1f}%')
