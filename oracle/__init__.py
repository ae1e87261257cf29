"""TEST INFRASTRUCTURE ONLY: the CPU oracle (restated reference API).  Imported by
tests/, __graft_entry__.smoke() and bench.py's CPU legs; never by the product."""
