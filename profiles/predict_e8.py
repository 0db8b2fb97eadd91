"""Predicted pipeline efficiency E(n) = T(1) / (n T(n)) of the C2 bench at n = 2, 4, 8 (m = 32,
except_last) from MEASURED n = 1 task times -- one B200 only in this run, so no scaling curve was
measured.  Model (clock-cycle schedule, Alg. 1, mirrored backward):

  T(n) = (m + n - 1) (t_F(n) + h) + (m + n - 1) (t_BF'(n) + h) + t_W / n + t_fold / n
  t_F(n)   = t_F(1) per block x (32 / n) + c   (c: per-task fixed cost = launch, first exchange, drain)
  t_BF'(n) = the paired B + F' task (both half grids, R5) per block x (32 / n) + c
  h        = per-clock hand-off: fused-send flag + the consumer's stream wait (one-way; half the CE
             ping-pong of profiles/round2_transport_sweep.txt as an upper bound)
c is fitted from the n = 1 phase timeline (F task = 64 phases x phase period + c).
    python profiles/predict_e8.py profiles/<round>/<bench>.json [phase_us]"""
import json
import sys

b = json.load(open(sys.argv[1]))
tasks = b["pipeline"]["tasks"]
m, blocks = 32, 32
T1 = b["ms_per_step"] * 1e3
tF1, tB1 = tasks["F"]["median_us"], tasks["B"]["median_us"]  # B = the paired B task (lane 0)
tW = tasks["W"]["median_us"]
phase = float(sys.argv[2]) if len(sys.argv) > 2 else 8.2  # measured F-task phase period (stamps)
c = max(tF1 - 2 * blocks * phase, 0.0)
fold = 450.0
h = 11.5 / 2  # one-way hand-off, CE ping-pong / 2 (the fused flag is cheaper)
print(f"n = 1 measured: T {T1 / 1e3:.2f} ms, F {tF1:.0f} us, paired B+F' {tB1:.0f} us, W+SGD {tW:.0f} us, c = {c:.0f} us")
for n in (2, 4, 8):
    tF = (tF1 - c) / n + c
    tB = (tB1 - c) / n + c
    T = (m + n - 1) * (tF + h) + (m + n - 1) * (tB + h) + tW / n + fold / n
    E = T1 / (n * T)
    Es = m / (m + n - 1)
    print(f"n = {n}: T {T / 1e3:6.2f} ms  {512 / (T * 1e-6):8.0f} samples/s  E {E:.3f}  E* {Es:.3f}  E/E* {E / Es:.3f}")
