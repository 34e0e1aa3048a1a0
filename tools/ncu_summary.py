"""Text summary of one kernel in an ncu report (--set full): headline
metrics, DRAM bytes, stall reasons and the hottest source lines."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, top=15):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, v = rows[0], rows[1], rows[2]
    print(f"report: {rep}")
    print(f"kernel: {v[h.index('Kernel Name')]}")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:62s} {v[i]:>18s} {units[i]}")
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
            try:
                st.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x[0] for x in st) or 1.0
    print("stall reasons (share of samples):")
    for x, n in sorted(st, reverse=True)[:8]:
        print(f"  {n:32s} {100 * x / tot:5.1f}%")
    src = ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    rows = list(csv.reader(io.StringIO(src)))
    hdr = next((r for r in rows if r and r[0] == "Line No"), None)
    if hdr:
        ws = hdr.index("Warp Stall Sampling (All Samples)")
        f, res = None, []
        for r in rows:
            if not r:
                continue
            if r[0] == "File Path":
                f = r[1].split("/")[-1]
                continue
            if r[0] in ("Function Name", "Line No") or r[0] == "":
                continue
            try:
                res.append((float(r[ws]), f, r[0], r[1].strip()[:90]))
            except (ValueError, IndexError):
                pass
        tw = sum(x[0] for x in res) or 1.0
        print("hottest source lines (share of stall samples):")
        for w, f, ln, s in sorted(res, reverse=True)[:top]:
            print(f"  {100 * w / tw:5.1f}%  {f}:{ln}  {s}")


if __name__ == "__main__":
    main(sys.argv[1])
