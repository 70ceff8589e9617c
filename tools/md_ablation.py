"""The md ablation: head-to-head self-play
on C3 rules (2p, 26 tiles with jokers, consecutive) of the paper's simplified
search (children keyed by the guess alone; flat UCT 64 x 1024) against
the vanilla tree keyed by (determinization, guess) at the SAME
playout budget per decision (1024 UCB iterations x 64 playouts), for a few
candidate-determinization counts.  Seats alternate over the same deals.
Reports the simplified search's win rate (95% interval) and the md root
fan-out (K determinizations x A guesses).

    python tools/md_ablation.py [games] [matchup indices, e.g. 3,4] > profiles/r01_md_ablation.jsonl
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    games = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    from paper_2403_10720_b200 import dvc
    from paper_2403_10720_b200.selfplay import play_games
    dvc.set_option("search_device", 1)
    fan = []

    def simplified(exp_n, n):
        def search(obs, s):
            best, _ = dvc.mcts_search(dvc.encode(obs), exp_n, n, s)
            return best
        return search

    def md(n_det):
        def search(obs, s):
            best, table, k = dvc.md_search(dvc.encode(obs), n_det, 1024, 64, s)
            fan.append(k * len(table))
            return best
        return search

    # (A name, A, B name, B): the keying at the paper's granularity (64 x 1024
    # against md's 1024 x 64), the keying alone at equal granularity, and the
    # granularity alone
    matchups = [("simplified flat 64x1024", simplified(64, 1024), "md n_det=%d, 1024x64" % k, md(k)) for k in (4, 16, 64)]
    matchups += [("simplified flat 1024x64", simplified(1024, 64), "md n_det=16, 1024x64", md(16)),
                 ("simplified flat 1024x64", simplified(1024, 64), "simplified flat 64x1024", simplified(64, 1024))]
    which = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else range(len(matchups))
    for mi in which:
        name_a, A, name_b, B = matchups[mi]
        fan.clear()
        t0 = time.perf_counter()
        res = []
        for half in (0, 1):
            def search(obs, s, half=half):
                return (A if obs["viewer"] == half else B)(obs, s)
            seeds = list(range(3000, 3000 + games // 2))
            out = play_games(seeds, threads=16, players=2, ranks=12, jokers=1, consecutive=1, per=4,
                             search=search)
            res += [1 if g["winner"] == half else 0 for g in out]
        w = sum(res)
        p = w / len(res)
        print(json.dumps({"a": name_a, "b": name_b, "games": len(res),
                          "a_wins": w, "a_win_rate": round(p, 4), "ci95": round(1.96 * math.sqrt(p * (1 - p) / len(res)), 4),
                          "md_root_children_mean": round(sum(fan) / max(1, len(fan)), 1) if fan else None,
                          "md_root_children_max": max(fan) if fan else None,
                          "playouts_per_decision": 65536, "s": round(time.perf_counter() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
