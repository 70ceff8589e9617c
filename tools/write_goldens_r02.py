"""Writes the round-2 hand-derived goldens (tests/golden/X3a.json, X4a.json,
J2.json, L1.json).  Every number below is derived by hand in the `derivation` field;
nothing here calls the oracle or the product (the tests check both against
these values, and tests/indep_exact.py re-derives them a second way)."""
import json, os

B = lambda v, r=False: {"color": "B", "value": v, "revealed": r}
W = lambda v, r=False: {"color": "W", "value": v, "revealed": r}
OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")

G = {
"X3a": {
 "citation": "PAPER:106 (a correct guess grants another attempt; the turn passes to the next gambler), PAPER:102 (last gambler standing); SPEC:186 round-robin turn order skipping eliminated players (SURVEY §8(c.7) #11, #20)",
 "rules": {"players": 3, "ranks": 2, "jokers": 0, "consecutive": 1},
 "viewer": 0,
 "lines": [[B(0, True), W(0)], [B(None)], [W(None)]],
 "pool_size": 0, "pending": -1, "correct_this_turn": 0,
 "expected": {"N": 1,
   "legal": [[1, 0, "B", 1], [2, 0, "W", 1]],
   "p_codes": [[1, 0, "B", 1], [2, 0, "W", 1]],
   "p_all": [["1/2", "0", "1/2"], ["1/2", "1/2", "0"]]},
 "derivation": (
  "R=2: keys B0 W0 B1 W1. U = T minus the viewer's {B0, W0} = {B1, W1}; seat 1's black slot must be B1 and seat 2's white slot W1, pool empty: N = 1. "
  "LEGAL(0) = seat 1 slot 0 black values not held/revealed = {B1}; seat 2 slot 0 white = {W1}. "
  "Action (1,0,B1): correct, seat 1 has no hidden tile (eliminated), seats 0 and 2 alive -> the viewer decides again (consecutive) with corr = 1: LEGAL = [(2,0,W1)] (seat 1 skipped: dead) + STOP, n = 2. "
  "Guess (1/2): correct, seat 2 eliminated, viewer wins. STOP (1/2): next mover after seat 0 is seat 1 -- dead, skipped -> seat 2; pool empty, no draw; "
  "seat 2's LEGAL = seat 0's hidden W0 slot (seat 1 dead) with white values not in {W1} nor revealed {B0, B1} = {W0}: correct, the viewer is eliminated, seat 2 wins. "
  "p = (1/2, 0, 1/2). Action (2,0,W1) is the mirror image: guess (1/2) viewer wins; STOP (1/2) -> seat 1 (alive) moves, its only guess is W0 at seat 0 (seat 2 dead) -> seat 1 wins: p = (1/2, 1/2, 0). "
  "Without skipping the dead seat, the STOP branch of (1,0,B1) would hand the move to seat 1, which has no hidden tile left.")
},
"J2": {
 "citation": "PAPER:102 (two jokers in the tile set), PAPER:104-106 (draw, a wrong guess reveals the newly drawn tile); joker reading SURVEY §8(c.7) #1 (a joker is a guessable value of its colour while unaccounted for)",
 "rules": {"players": 2, "ranks": 2, "jokers": 1, "consecutive": 1},
 "viewer": 0,
 "lines": [[B(0), W(1)], [W(0, True), B(None)]],
 "pool_size": 2, "pending": 1, "correct_this_turn": 1,
 "expected": {"N": 2,
   "legal": [[1, 1, "B", 1], [1, 1, "B", "J"], "STOP"],
   "p_codes": [[1, 1, "B", 1], [1, 1, "B", "J"]],
   "p_all": [["5/8", "3/8"], ["5/8", "3/8"]]},
 "derivation": (
  "R=2 with jokers: keys B0 W0 B1 W1 JB JW. Viewer [B0, W1 (pending)], all hidden; opponent [W0 revealed, B?]. U = {B1, JB, JW}. "
  "The black slot right of W0 holds B1 (order W0 < B1 holds) or JB (jokers carry no order); the other two tiles are the pool: N = 2, each 1/2. "
  "LEGAL(0) = values of the black slot not held/revealed = {B1, JB}, then STOP (corr = 1). "
  "Action (1,1,B1): correct (slot = B1, 1/2) -> opponent has no hidden tile -> viewer wins. Wrong (slot = JB, 1/2): the viewer reveals its pending W1 (B0 still hidden); "
  "the opponent draws from pool {B1, JW}. Draws B1 (1/2): its guess at the viewer's B0 slot lists black values not in {W0, JB, B1} and not revealed = {B0} -> correct -> viewer eliminated. "
  "Draws JW (1/2; any gap): the list is {B0, B1} (JB is its own). B0 (1/2) -> viewer eliminated. B1 (1/2) -> wrong -> the opponent reveals its drawn JW (not JB); "
  "viewer's turn: draws B1 (last pool tile); its only guess at the opponent's hidden black slot is JB (B0, B1 its own) -> correct -> viewer wins. "
  "Continuation = 1/2*0 + 1/2*(1/2*0 + 1/2*1) = 1/4; p = 1/2 + 1/2*1/4 = 5/8. "
  "Action (1,1,JB): correct (slot = JB) -> win; wrong (slot = B1): viewer reveals W1, the opponent draws from {JB, JW}: JB (1/2) -> its list for the B0 slot is {B0} -> viewer eliminated; "
  "JW (1/2) -> list {B0, JB}: B0 (1/2) loses; JB (1/2) is wrong -> opponent reveals its drawn JW; viewer draws JB (any gap) and its only guess at the opponent's black slot is B1 -> correct -> win. "
  "p = 1/2 + 1/2*1/4 = 5/8. (STOP's value 11/18 comes from the two enumerators, not derived by hand.)")
},
"L1": {
 "citation": "SPEC:184 (a wrong guess with nothing drawn reveals the guesser's leftmost hidden tile; SURVEY §8(c.7) #8, the empty-pool reading), PAPER:106 (one reveal per wrong guess), PAPER:153 (consecutive = 0: one guess per turn)",
 "rules": {"players": 2, "ranks": 3, "jokers": 0, "consecutive": 0},
 "viewer": 0,
 "lines": [[B(0), B(1), W(2)], [W(None), W(None), B(None)]],
 "pool_size": 0, "pending": -1, "correct_this_turn": 0,
 "expected": {"N": 1,
   "legal": [[1, 0, "W", 0], [1, 0, "W", 1], [1, 1, "W", 0], [1, 1, "W", 1], [1, 2, "B", 2]],
   "p_codes": [[1, 0, "W", 0], [1, 0, "W", 1], [1, 1, "W", 0], [1, 1, "W", 1]],
   "p_all": [["1", "0"], ["0", "1"], ["0", "1"], ["1", "0"]]},
 "derivation": (
  "R=3: keys B0 W0 B1 W1 B2 W2. Viewer [B0, B1, W2] all hidden, opponent [W?, W?, B?], pool empty (pending -1). U = {W0, W1, B2}: "
  "colours force the black slot to B2 and the ascending order forces W0 < W1: N = 1, opponent line [W0, W1, B2]. LEGAL(0): white slots list {W0, W1} each, the black slot {B2}. "
  "Action (1,0,W1), wrong: nothing was drawn, so the viewer reveals its LEFTMOST hidden tile B0 and keeps B1, W2; the opponent keeps 3 hidden. "
  "From here every opponent guess is forced and correct: its list for the B1 slot is the black values not in {W0, W1, B2} and not revealed {B0} = {B1}, for the W2 slot {W2}, "
  "and after one of them is revealed the other list is unchanged. One guess per turn (consecutive = 0): the opponent needs 2 hits and moves first, the viewer needs 3 hits "
  "(and a wrong viewer guess reveals its own tile): opponent hit, viewer's one guess, opponent hit -> the viewer is eliminated first. p = 0. "
  "(Revealing the RIGHTMOST hidden tile W2 instead would leave {B0, B1}, where the opponent's list is {B0, B1} for each slot and it can miss, so p > 0: "
  "the golden separates the two readings.) Action (1,1,W0) is the same wrong guess at the other white slot: p = 0. "
  "Action (1,0,W0), correct: W0 revealed, the opponent keeps W1, B2 hidden; the viewer keeps 3. From here every viewer guess is forced and correct "
  "(its list for the W1 slot is {W1}: W0 revealed, W2 its own; for the B2 slot {B2}: B0, B1 its own). The viewer needs 2 hits, the opponent 3, one guess per turn, "
  "the opponent moving first: opponent guess, viewer hit, opponent guess, viewer hit -> the opponent is out first (an opponent miss only reveals its own tile). p = 1. "
  "(1,1,W1) is the same correct guess: p = 1. "
  "((1,2,B2)'s 7/10 comes from the enumerators.)")
},
"X4a": {
 "citation": "PAPER:106 (the turn passes to the next gambler; a correct guess grants another attempt), PAPER:102 (last gambler standing); SPEC:186 round-robin skipping eliminated players -- here two in a row (SURVEY §8(c.7) #11)",
 "rules": {"players": 4, "ranks": 3, "jokers": 0, "consecutive": 1},
 "viewer": 0,
 "lines": [[B(0, True), W(0)], [B(1, True)], [W(1, True)], [B(None), W(None)]],
 "pool_size": 0, "pending": -1, "correct_this_turn": 0,
 "expected": {"N": 1,
   "legal": [[3, 0, "B", 2], [3, 1, "W", 2]],
   "p_codes": [[3, 0, "B", 2], [3, 1, "W", 2]],
   "p_all": [["1/2", "0", "0", "1/2"], ["1/2", "0", "0", "1/2"]]},
 "derivation": (
  "R=3: keys B0 W0 B1 W1 B2 W2. Seats 1 [B1] and 2 [W1] have every tile revealed: both are already eliminated. "
  "U = T minus the viewer's {B0, W0} and the revealed {B1, W1} = {B2, W2}: seat 3's black slot is B2, its white slot W2, pool empty: N = 1. "
  "LEGAL(0): seats 1 and 2 are skipped (dead); seat 3's black slot lists black values not held/revealed = {B2}, its white slot {W2}. "
  "Action (3,0,B2): correct; seat 3 keeps W2, the viewer keeps W0, so two players are alive and the viewer decides again (consecutive) with "
  "LEGAL = [(3,1,W2)] + STOP, n = 2. Guess (1/2): correct, seat 3 eliminated, the viewer wins. STOP (1/2): the next mover after seat 0 is seat 1 "
  "-- dead -- then seat 2 -- dead -- then seat 3; no draw (pool empty); seat 3's only target is the viewer's hidden W0 slot, whose list is the white "
  "values not in {B2, W2} and not revealed {B0, B1, W1} = {W0}: correct, the viewer is eliminated, seat 3 wins. p = (1/2, 0, 0, 1/2). "
  "Action (3,1,W2) is the mirror image (guess B2 next, or STOP): p = (1/2, 0, 0, 1/2). "
  "Handing the move to a dead seat instead (no skipping) would make seat 1, which has no hidden tile, move.")
},
}

for name, d in G.items():
    with open(os.path.join(OUT, name + ".json"), "w") as f:
        json.dump(d, f, indent=1)
        f.write("\n")
print("wrote", ", ".join(G))
