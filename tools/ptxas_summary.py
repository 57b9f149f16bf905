"""Summarise `ptxas -v` of the hot kernels from paper_1511_07983_b200/build.log.

    python tools/ptxas_summary.py > profiles/r02_ptxas.txt
"""
import os
import re
import sys

LOG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1511_07983_b200", "build.log")
# (kernel, mangled template-args suffix) for C4's variant (S' = 2, full) and the policy/direct kernels
WANT = [
    ("rk_dp_levels_coop_kernel", "ILi2ELb1E", "<2,true>"),
    ("rk_dp_level_kernel", "ILi2ELb1E", "<2,true>"),
    ("rk_dp_small_levels_kernel", "ILi2ELb1E", "<2,true>"),
    ("rk_dp_keys32_kernel", "ILj8E", "<8>"),
    ("rk_dp_suffix_kernel", "ILi2ELb1E", "<2,true>"),
    ("rk_dp_row24_kernel", "ILi2ELb1E", "<2,true>"),
    ("rk_eval_kernel", "ILi2ELb1E", "<2,true>"),
    ("rk_batch_kernel", "ILi2ELb1E", "<2,true>"),
    ("rk_policy_eval_kernel", "ILi2E", "<2>"),
    ("rk_dp_keys_kernel", "", ""),
    ("rk_dp_rows_kernel", "", ""),
    ("rk_dp_ext_kernel", "", ""),
    ("rk_dp_children_kernel", "", ""),
    ("rk_dp_parents_kernel", "", ""),
    ("rk_dp_runs_kernel", "", ""),
]


def main():
    lines = open(LOG).read().split("\n")
    print("ptxas -v (sm_100a) of the memoised step's kernels for C4's variant (2 super-SMs) and the policy/direct kernels")
    for name, targs, label in WANT:
        pat = re.compile(r"Compiling entry function '_Z\S*\d" + name + (targs if targs else r"(?:E|v|P)"))
        for i, l in enumerate(lines):
            if pat.search(l):
                tag = f"{name} {label}".ljust(38)
                print(tag, lines[i + 2].strip())
                print(tag, lines[i + 3].strip())
                break
        else:
            print(f"{name} {label}".ljust(38), "not found", file=sys.stderr)


if __name__ == "__main__":
    main()
