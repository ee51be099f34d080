"""One line per ncu report: duration, L2->L1 read rate, L1/L2/DRAM
throughput, issue, occupancy, registers, LSU wavefronts (global / shared).

    python tools/ncu_brief.py gpurun_out/x.ncu-rep [...]"""
import csv
import io
import subprocess
import sys


def brief(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))

    def g(k):
        try:
            return float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")

    scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
    sec = g("gpu__time_duration.sum") * scale.get(u.get("gpu__time_duration.sum", "ns"), 1e-9)
    xbar = g("l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum") * 32
    return (f"{path.split('/')[-1]:28s} {d.get('Kernel Name', '')[:44]:44s} {sec * 1e3:8.3f} ms  "
            f"xbar->L1 {xbar / sec / 1e12:5.2f} TB/s  L1 {g('l1tex__throughput.avg.pct_of_peak_sustained_active'):5.1f}%  "
            f"L2 {g('lts__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}%  "
            f"DRAM {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}%  "
            f"issue {g('smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f}%  "
            f"warps {g('sm__warps_active.avg.per_cycle_active'):5.1f}  regs {d.get('launch__registers_per_thread')}  "
            f"glb-ld wf {g('l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum'):.3g}  "
            f"shared wf {g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum'):.3g}  "
            f"inst {g('smsp__inst_executed.sum'):.3g}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(brief(p))
