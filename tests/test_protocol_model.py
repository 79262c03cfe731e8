"""Exhaustive interleavings of the engine's round protocol (tests/protocol_model.py):
P=2 controllers section by section, owners' done words, back-to-back offers
and a host reader's pin handshake.  The shipped protocol is clean; the
variants that are not -- the pre-fix publication order, a reader assuming
the wrong lead -- are caught."""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import protocol_model as M  # noqa: E402


def test_two_rounds_in_flight_protocol_is_clean():
    rep = M.explore(p=2, rounds=4, R=3, lead=2, preposted=True)
    assert rep.ok, rep.violations[:1]
    assert rep.states > 100_000 and rep.terminals > 100


def test_one_round_in_flight_protocol_is_clean():
    rep = M.explore(p=2, rounds=4, R=2, lead=1, preposted=True)
    assert rep.ok, rep.violations[:1]


def test_explorer_finds_the_publication_race_the_fix_closed():
    """Acknowledging a host pin before publishing a completed round lets the
    reader pin a slot round G + R is already writing (fixed in the controller:
    publish_host() before the ack)."""
    rep = M.explore(p=2, rounds=4, R=3, lead=2, preposted=True, ack_publishes=False)
    assert rep.violations and rep.violations[0][0] == "pinned slot overwritten"


def test_explorer_finds_a_wrong_reader_margin():
    """With two rounds in flight a reader must re-check with the two-round
    margin (done + 2 < G + R, ec_wait / wait_and_pin); the one-round margin
    is unsafe.  (Two in flight on two slots is refused by construction:
    EcDesc::lead is 2 only with R >= 3.)"""
    rep = M.explore(p=2, rounds=4, R=3, lead=2, preposted=True, reader_lead=1)
    assert rep.violations and rep.violations[0][0] == "pinned slot overwritten"
