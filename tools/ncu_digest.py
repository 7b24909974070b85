"""Digest of an ncu --set full report: per kernel, the headline metrics, top stall reasons and
the source lines with the most warp-stall samples. Usage: python tools/ncu_digest.py rep [regex]"""
import csv
import io
import re
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'smsp__inst_executed.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active']


def ncu(*args):
    return subprocess.run(['ncu', *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rx = sys.argv[2] if len(sys.argv) > 2 else '.'
    rows = list(csv.reader(io.StringIO(ncu('-i', rep, '--page', 'raw', '--csv'))))
    hdr, units = rows[0], rows[1]
    for idx, r in enumerate(rows[2:]):
        name = r[hdr.index('Kernel Name')]
        if not re.search(rx, name):
            continue
        print('==', name[:110])
        for w in WANT:
            if w in hdr:
                print(f"  {w:62s} {r[hdr.index(w)]} {units[hdr.index(w)]}")
        st = []
        for i, h in enumerate(hdr):
            if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued'):
                try:
                    st.append((float(r[i].replace(',', '')), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        st.sort(reverse=True)
        tot = sum(v for v, _ in st) or 1
        print('  stalls:', ', '.join(f"{h} {v / tot * 100:.0f}%" for v, h in st[:7]))
        kname = re.sub(r'\(.*', '', name).split('::')[-1].split('<')[0]
        # this launch only (a name regex would merge template instantiations)
        src = list(csv.reader(io.StringIO(ncu('-i', rep, '--page', 'source', '--csv', '--launch-skip', str(idx),
                                              '--launch-count', '1', '--print-source', 'cuda,sass'))))
        out, fname = [], ''
        for s in src:
            if len(s) >= 2 and s[0] == 'File Path':
                fname = s[1].split('/')[-1]
            if len(s) > 7 and s[0].isdigit():
                try:
                    out.append((float(s[4]), float(s[7]), fname, s[0], s[1][:80]))
                except ValueError:
                    pass
        tot = sum(o[0] for o in out) or 1
        for o in sorted(out, reverse=True)[:14]:
            print(f"  {o[0] / tot * 100:5.1f}% inst {o[1] / 1e3:7.0f}k {o[2]}:{o[3]} {o[4]}")


if __name__ == '__main__':
    main()
