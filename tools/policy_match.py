"""Head-to-head self-play (C3 rules: 2p, 26 tiles with jokers, consecutive):
seat A searches with one batch variant, seat B with another; seats alternate
game by game.  Reports A's win rate with a 95% interval.  Measures what the
N4 variants (DESIGN.md §R3 CRN, §R10 informed policy) do to playing strength.

    python tools/policy_match.py [games] [expansions] [sims_per_child]
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
    exp_n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
    from paper_2403_10720_b200 import dvc
    from paper_2403_10720_b200.selfplay import play_games
    dvc.set_option("search_device", 1)

    def agent(crn, informed):
        def search(obs, s):
            st = dvc.encode(obs)
            best, _ = dvc.mcts_search(st, exp_n, n, s, crn=crn, informed=informed)
            return best
        return search

    matchups = [("informed", (False, True), "plain", (False, False)),
                ("crn", (True, False), "plain", (False, False)),
                ("informed+crn", (True, True), "informed", (False, True))]
    for name_a, fa, name_b, fb in matchups:
        A, B = agent(*fa), agent(*fb)
        t0 = time.perf_counter()
        res = []
        for half in (0, 1):
            # A sits at seat `half` in every game of this half
            def search(obs, s, half=half):
                return (A if obs["viewer"] == half else B)(obs, s)
            seeds = list(range(1000, 1000 + games // 2))          # the same deals with seats swapped
            out = play_games(seeds, threads=16, players=2, ranks=12, jokers=1, consecutive=1, per=4,
                             search=search)
            res += [1 if g["winner"] == half else 0 for g in out]
        w = sum(res)
        p = w / len(res)
        ci = 1.96 * math.sqrt(p * (1 - p) / len(res))
        print(json.dumps({"a": name_a, "b": name_b, "games": len(res), "a_wins": w, "a_win_rate": round(p, 4),
                          "ci95": round(ci, 4), "expansions": exp_n, "sims_per_child": n,
                          "s": round(time.perf_counter() - t0, 1)}), flush=True)


if __name__ == "__main__":
    main()
