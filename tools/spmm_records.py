#!/usr/bin/env python
"""`spmm_cli bench` on the B200: JSON-lines records and the reference's CSV
(paper_2007_03179_b200.records; spmm_cli.cpp:566-611).

    python tools/spmm_records.py --gen ROWS,NNZ,SEED | --csr1 PATH
        [--n 32,64,128] [--variants naive,crc,crc-cwm,tuned] [--cf 2] [--op sum]
        [--repeats 9] [--b-seed 42] [--verify] [--jsonl out.jsonl] [--csv out.csv]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2007_03179_b200 as G
    from paper_2007_03179_b200 import records as R

    p = argparse.ArgumentParser()
    src = p.add_mutually_exclusive_group(required=True)
    src.add_argument("--gen", help="ROWS,NNZ,SEED: gen_uniform_random (generate.hpp:39-69)")
    src.add_argument("--csr1", help="CSR1 cache file (io.hpp:15-16)")
    p.add_argument("--n", default="32,64,128")
    p.add_argument("--variants", default="naive,crc,crc-cwm,tuned")
    p.add_argument("--cf", type=int, default=2)
    p.add_argument("--op", default="sum")
    p.add_argument("--repeats", type=int, default=9)
    p.add_argument("--b-seed", type=int, default=42)
    p.add_argument("--verify", action="store_true")
    p.add_argument("--jsonl", default=None)
    p.add_argument("--csv", default=None)
    args = p.parse_args()
    gen = None
    if args.gen:
        rows, nnz, seed = (int(x) for x in args.gen.split(","))
        a = G.gen_uniform_random(G.GraphGenSpec(rows, nnz, seed))
        gen = {"rows": rows, "nnz": nnz, "seed": seed, "self_loops": False}
        desc = f"gen:{rows},{nnz},{seed}"
    else:
        a = G.read_csr_cache(args.csr1)
        desc = args.csr1
    variants = [G.variant_by_name(v, args.cf) for v in args.variants.split(",")]
    jf = open(args.jsonl, "w") if args.jsonl else sys.stdout
    reference = None
    if args.verify:  # the CPU oracle as the checker (test infrastructure)
        import oracle as O

        def reference(m, b, op):
            return O.spmm(m.n_rows, m.n_cols, m.row_ptr, m.col_ind, m.vals, b.data, op)[0]
    rows = []
    for rec, line in R.bench_records(a, desc, [int(x) for x in args.n.split(",")], variants,
                                     args.op, args.repeats, args.b_seed, gen, reference):
        jf.write(R.dumps(rec) + "\n")
        jf.flush()
        rows.append(line)
    if args.csv:
        with open(args.csv, "w") as f:
            f.write(R.CSV_HEADER + "\n")
            for line in rows:
                f.write(line + "\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
