"""Run the reference's harness entry points on the device (bench_recon / profile_breakdown)
for a BASELINE config and print the text reports:  python tools/harness_demo.py [n M Q it]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_10928_b200 as pk  # noqa: E402

n, M, Q, it = (int(v) for v in (sys.argv[1:5] if len(sys.argv) >= 5 else (128, 128, 1024, 10)))
print(pk.bench_recon(n, M, Q, pk.ReconConfig(iterations=it), reps=5).to_text())
print(pk.profile_breakdown(n, M, Q, pk.ReconConfig(iterations=it)).to_text())
