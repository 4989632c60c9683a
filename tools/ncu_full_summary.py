"""Key metrics of one `ncu --set full` capture (the dominant kernel) as markdown.

    ncu -i gpurun_out/X.ncu-rep --page raw --csv > /tmp/raw.csv
    python tools/ncu_full_summary.py /tmp/raw.csv "title" [algorithmic_bytes] > profiles/r01_X.md
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "kernel time"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active", "tensor HMMA subpipe active %"),
    ("sm__ops_path_tensor_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed", "tf32 tensor ops % of peak"),
    ("sm__ops_path_tensor_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed", "bf16 tensor ops % of peak"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "TMEM active %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "smem wavefronts, tensor-core operand reads"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem wavefronts, LSU loads"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem wavefronts, LSU stores"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem bank conflicts, loads"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smem bank conflicts, stores"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(path, title, algo_bytes=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"# {title}\n\nkernel: `{name[:160]}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        got = {}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                got[key] = (vals[i], units[i])
                print(f"| {label} (`{key}`) | {vals[i]} | {units[i]} |")
        if algo_bytes and "dram__bytes_read.sum" in got:
            def mb(k):
                v, u = got[k]
                v = float(v.replace(",", ""))
                return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            traffic = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
            print(f"\nDRAM traffic {traffic:.1f} MB per launch vs {float(algo_bytes) / 1e6:.1f} MB algorithmic "
                  f"({traffic / (float(algo_bytes) / 1e6):.2f}x)")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
