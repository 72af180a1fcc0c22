"""Dump the encoded device plan of a config: passes, gate groups, sub-ops, diag term counts."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2008_00216_b200 as stv
from inputs import circuits as C
from tests import blob_emu as B
c=C.config(int(sys.argv[1]) if len(sys.argv)>1 else 2)
blob,offs=stv.plan_blob(c.n,c.gates)
for pi,po in enumerate(offs):
  P=B._at(blob,B.Pass,po)
  print('pass',pi,'kind',P.kind,'S',P.S,'L',P.L,'h',P.h,'hpos',list(P.hpos)[:P.h],'nops',P.nops,'ntab',P.ntab,'rec',P.rec_bytes)
  if not P.grouped: continue
  for i in range(P.nops):
    op=B._at(blob,B.Group,po+P.ops_off+256*i)
    s=[]
    for k in range(op.nsub):
      sb=B._at(blob,B.Sub,po+op.sub_off+16*k)
      c=sb.code&0xff
      if c<4: s.append('U1(%d)'%c)
      elif c<10: s.append('U2(%d%d)'%B.U2_PAIRS[c-4])
      elif c>=48: s.append('U2R(%d%d)'%B.U2_PAIRS[c-48])
      elif c>=44: s.append('U1R(%d)'%(c-44))
      elif c>=41: s.append('U2x2%d'%(c-41))
      elif c>=37: s.append('DH%d(m%d)'%(c-37,B._at(blob,B.DTab,po+P.tab_off+48*sb.arg).m))
      elif c>=31: s.append('U2V(%d%d;%d)'%(B.U2_PAIRS[c-31]+(sum(((sb.code>>(8+5*i))&31)!=31 for i in range(3)),)))
      elif c<30: s.append('CX(%d,%d%s%s)'%((c-10)//4-1,(c-10)%4,',raw%d'%(sb.ctl&0xffff) if sb.ctl&0xffff else '',',p%d'%((sb.ctl>>16)-1) if sb.ctl>>16 else ''))
      else:
        d=B._at(blob,B.DTab,po+P.tab_off+48*sb.arg)
        s.append('D(m%d,t%d)'%(d.m,d.nterm))
    print('  grp',list(op.tpos),' '.join(s))
  if P.ntc:
    for i in range(P.ntc):
      s=B._at(blob,B.TcStep,po+P.tc_off+32*i)
      print('    tc step', i, 'grp', s.group, 'M' if s.kind else 'E', 'subs[%d:%d]'%(s.first,s.first+s.n), 'op', s.op, 'dep 0x%x'%s.dep, 'bvar', s.bvar, 'last' if s.last else '')
